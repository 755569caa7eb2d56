"""Input generator checks (ndgi_synth) and the paper's BPP tables.

The BPP test pins the storage formats chosen for Theta (BC7 8 bits/texel for
F_uv and each F_uvt slice, raw u8 line maps, f16 MLP weights; reading R11) to
the numbers the paper prints in Table 2 and Table 3,
fixture tests/golden/paper_bpp.txt.
"""
import os

import numpy as np
import pytest

import ndgi_synth as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_bpp.txt")


def _rows():
    for line in open(GOLDEN):
        if line.strip() and not line.startswith("#"):
            name, prof, fmt, bpp, *_ = line.split()
            yield name, prof, fmt, float(bpp)


@pytest.mark.parametrize("name,prof,fmt,bpp", list(_rows()))
def test_bpp_matches_paper_tables(name, prof, fmt, bpp):
    # Table 1 set: 26 lightmaps of 128^2, one tile of 128^2
    lay = S.layout(1, 1, 1, prof, fmt_uv=fmt, fmt_uvt=fmt, fmt_line="u8" if fmt == "bc7" else fmt)
    got = S.theta_bytes(lay) * 8 / (26 * 128 * 128)
    assert abs(got - bpp) / bpp < 0.02, (name, got, bpp)


def test_deterministic_and_shardable():
    lay, seed = S.config("c2")
    a = S.make_theta(lay, seed, tiles=[3, 700, 1023])
    b = S.make_theta(lay, seed, tiles=[700])
    for k in a:
        np.testing.assert_array_equal(a[k][1], b[k][0])
    c = S.make_theta(lay, seed, tiles=[3, 700, 1023])
    for k in a:
        np.testing.assert_array_equal(a[k], c[k])


def test_shapes_and_modes():
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed)
    assert th["uv"].shape == (4, 32, 32, 16) and th["uvt"].shape == (4, 4, 8, 8, 16)
    assert th["ut"].shape == (4, 4, 64, 2) and th["mlp"].shape == (4, 595)
    assert ((th["uv"][..., 0] & 0x7F) == 0x40).all()          # smooth payload = mode 6
    mixed = S.make_theta(lay, seed, "mixed")["uv"][..., 0]
    modes = np.array([(int(b) & -int(b)).bit_length() - 1 for b in mixed.ravel()])
    assert set(modes.tolist()) == set(range(8))


def test_vt_batches_distinct():
    for ids, t in S.vt_batches(16384, 512, 3):
        assert len(set(ids.tolist())) == 512 and 0 <= t < 1
