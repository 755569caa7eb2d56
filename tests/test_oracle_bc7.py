"""Pins for the oracle's BC7 decoder (oracle/ndgi_oracle.c).

The paper stores F_uv and every t-slice of F_uvt as BC7 and
relies on the hardware decoder.  The oracle's scalar decoder is pinned
to things other than itself:
* Pillow 12.2.0's independent BCn decoder (mode 7 = BC7) on random blocks of
  every mode 0..7 (mode 8 excluded: reading R9, Pillow deviates from D3D);
* hand vectors (tests/golden/bc7_vectors.txt) with closed-form expectations;
* structural invariants of the format (bit budgets, weight tables, anchors).
"""
import os

import numpy as np
import pytest
from PIL import Image

import ndgi_synth as S
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "bc7_vectors.txt")


def _golden():
    out = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        hexblk, *texels = line.split()
        exp = np.array([[int(c) for c in t.split(",")] for t in texels], np.uint8)
        out.append((bytes.fromhex(hexblk), exp))
    return out


@pytest.mark.parametrize("blk,exp", _golden())
def test_golden_vectors(blk, exp):
    got, _ = oracle.bc7_decode_block(blk)
    np.testing.assert_array_equal(got, exp)


def _pillow(blocks, w, h):
    return np.asarray(Image.frombytes("RGBA", (w, h), np.ascontiguousarray(blocks).tobytes(), "bcn", 7))


@pytest.mark.parametrize("mode", range(8))
def test_against_pillow_random_blocks(mode):
    # 2^16 random blocks of one mode in a 1024x1024 image
    n = 256 * 256
    words = S.splitmix64(np.arange(2 * n, dtype=np.uint64) + np.uint64(1_000_003 * (mode + 1))).reshape(n, 2)
    blocks = S.bc7_random_blocks(words, np.full(n, mode))
    got = oracle.bc7_decode_image(blocks, 1024, 1024)
    np.testing.assert_array_equal(got, _pillow(blocks, 1024, 1024))


def test_against_pillow_mixed_and_smooth_payloads():
    lay, seed = S.config("c1")
    for payload in ("smooth", "mixed"):
        th = S.make_theta(lay, seed, payload)
        blocks = th["uv"].reshape(-1, 16)          # 4 tiles x 1024 blocks -> 256x256 image
        got = oracle.bc7_decode_image(blocks, 256, 256)
        np.testing.assert_array_equal(got, _pillow(blocks, 256, 256))
        sl = th["uvt"].reshape(-1, 16)             # 4 tiles x 4 slices x 64 blocks
        got = oracle.bc7_decode_image(sl, 64, 64)
        np.testing.assert_array_equal(got, _pillow(sl, 64, 64))


def test_mode8_is_zero_and_differs_from_pillow():
    blk = bytes(16)
    got, nbits = oracle.bc7_decode_block(blk)
    assert (got == 0).all()
    pil = _pillow(np.frombuffer(blk, np.uint8), 4, 4).reshape(16, 4)
    assert (pil[:, 3] == 255).all()   # the documented Pillow deviation (R9)


@pytest.mark.parametrize("mode", range(8))
def test_bit_budget_is_128(mode):
    # every field of every mode is consumed exactly once: the reader ends at bit 128
    n = 64
    words = S.splitmix64(np.arange(2 * n, dtype=np.uint64) + np.uint64(77 + mode)).reshape(n, 2)
    for b in S.bc7_random_blocks(words, np.full(n, mode)):
        assert oracle.bc7_decode_block(b.tobytes())[1] == 128


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_weight_tables_closed_form(bits):
    for i in range(1 << bits):
        assert oracle.bc7_weight(bits, i) == int(np.floor(64 * i / ((1 << bits) - 1) + 0.5))


def test_partition_tables_structure():
    for p in range(64):
        assert oracle.bc7_subset(2, p, 0) == 0 and oracle.bc7_subset(3, p, 0) == 0
        a = oracle.bc7_anchor(2, p, 1)
        assert oracle.bc7_subset(2, p, a) == 1
        for s in (1, 2):
            assert oracle.bc7_subset(3, p, oracle.bc7_anchor(3, p, s)) == s
        # every subset is populated
        assert {oracle.bc7_subset(2, p, i) for i in range(16)} == {0, 1}
        assert {oracle.bc7_subset(3, p, i) for i in range(16)} == {0, 1, 2}


def _pack(fields):
    v, pos = 0, 0
    for val, w in fields:
        v |= (val & ((1 << w) - 1)) << pos
        pos += w
    assert pos == 128
    return v.to_bytes(16, "little")


def test_pbit_and_expansion_semantics():
    # mode 3 (2 subsets, 7-bit RGB, one p-bit per endpoint), partition 0:
    # R = 127 with p = 1 -> 255 ; G = B = 0 with p = 1 -> 1  (D3D11: p-bit is the LSB)
    f = [(1 << 3, 4), (0, 6)]
    f += [(127, 7)] * 4 + [(0, 7)] * 8          # R for 4 endpoints, then G, B
    f += [(1, 1)] * 4                           # p-bits
    f += [(0, 30)]                              # indices all zero -> texels = e0 of their subset
    got, n = oracle.bc7_decode_block(_pack(f))
    assert n == 128
    assert (got[:, 0] == 255).all() and (got[:, 1] == 1).all() and (got[:, 2] == 1).all() and (got[:, 3] == 255).all()
    # 7-bit 10 with p = 0 -> 20 (mode 6)
    f = [(1 << 6, 7)] + [(10, 7)] * 8 + [(0, 1), (0, 1), (0, 63)]
    got, _ = oracle.bc7_decode_block(_pack(f))
    assert (got == 20).all()


def test_rotation_and_index_select():
    # mode 5, rotation 1 swaps R and A: colour 20, alpha 255 -> (255, 20, 20, 20)
    f = [(1 << 5, 6), (1, 2)] + [(10, 7)] * 6 + [(255, 8)] * 2 + [(0, 31), (0, 31)]
    got, n = oracle.bc7_decode_block(_pack(f))
    assert n == 128
    assert (got == np.array([255, 20, 20, 20], np.uint8)).all()
    # mode 4: colour endpoints 0 -> 31 (5-bit), alpha 0 -> 63 (6-bit); texel 1 index 1 in both arrays.
    # select 0: colour uses 2-bit weights (w=21 -> 84), alpha the 3-bit (w=9 -> 36)
    for isel, exp in ((0, (84, 84, 84, 36)), (1, (36, 36, 36, 84))):
        f = [(1 << 4, 5), (0, 2), (isel, 1)] + [(0, 5), (31, 5)] * 3 + [(0, 6), (63, 6)]
        f += [(0, 1), (1, 2)] + [(0, 2)] * 14      # primary (2-bit), texel 0 anchor has 1 bit
        f += [(0, 2), (1, 3)] + [(0, 3)] * 14      # secondary (3-bit)
        got, n = oracle.bc7_decode_block(_pack(f))
        assert n == 128
        assert tuple(got[1]) == exp, (isel, got[1])
