"""Pins for gamma(t) (Eq. 4) and the decoder MLP G_Phi.

gamma: closed-form values.  GELU: closed-form values of both variants (the
erf value at 3 is 2.995950, the tanh value 2.996363; SURVEY.md notes that
SPEC.md S:240 mislabels the erf value).  MLP: torch fp64 F.linear + F.gelu,
an independent library implementation of the same layers.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import ndgi_synth as S
import oracle


def test_gamma_closed_forms():
    np.testing.assert_allclose(oracle.gamma(0.0), [0, 1, 0, 1], atol=1e-15)
    np.testing.assert_allclose(oracle.gamma(0.5), [1, 0, 0, -1], atol=1e-15)
    r = math.sqrt(2) / 2
    np.testing.assert_allclose(oracle.gamma(0.25), [r, r, 1, 0], atol=1e-15)
    np.testing.assert_allclose(oracle.gamma(1.0), [0, -1, 0, 1], atol=1e-15)  # not 1-periodic (R4)


def test_gelu_values():
    assert abs(oracle.gelu(3.0, "erf") - 2.9959502) < 1e-6
    assert abs(oracle.gelu(3.0, "tanh") - 2.9963627) < 1e-6
    assert oracle.gelu(0.0, "erf") == 0.0
    for z in np.linspace(-6, 6, 97):
        tz = torch.tensor([z], dtype=torch.float64)
        assert abs(oracle.gelu(z, "erf") - F.gelu(tz).item()) < 1e-15
        assert abs(oracle.gelu(z, "tanh") - F.gelu(tz, approximate="tanh").item()) < 1e-15
    # the two variants differ by at most ~4.73e-4
    zs = np.linspace(-8, 8, 16001)
    d = max(abs(oracle.gelu(z, "erf") - oracle.gelu(z, "tanh")) for z in zs)
    assert 4.6e-4 < d < 4.8e-4


@pytest.mark.parametrize("h,variant", [(16, "erf"), (16, "tanh"), (64, "erf"), (8, "tanh")])
def test_mlp_vs_torch(h, variant):
    lay = S.layout(1, 4, 1, "M", hidden=h)
    w = S.make_theta(lay, 11 + h)["mlp"]
    rng = np.random.default_rng(h)
    for k in range(4):
        wk = w[k].view(np.float16).astype(np.float64)
        W1 = wk[:16 * h].reshape(h, 16); o = 16 * h
        b1 = wk[o:o + h]; o += h
        W2 = wk[o:o + h * h].reshape(h, h); o += h * h
        b2 = wk[o:o + h]; o += h
        W3 = wk[o:o + 3 * h].reshape(3, h); o += 3 * h
        b3 = wk[o:o + 3]
        approx = "none" if variant == "erf" else "tanh"
        x = rng.uniform(0, 1, (8, 16))
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        ref = F.linear(F.gelu(F.linear(F.gelu(F.linear(T(x), T(W1), T(b1)), approximate=approx), T(W2), T(b2)),
                              approximate=approx), T(W3), T(b3)).numpy()
        got = np.array([oracle.mlp(h, w[k], x[i], variant) for i in range(8)])
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13)


def test_mlp_param_count_and_zero_weights():
    assert oracle.mlp_params(16) == 595
    assert oracle.mlp_params(64) == 5443
    h = 16
    w = np.zeros(595, np.float16)
    w[-3:] = [0.25, 0.5, 0.75]
    y = oracle.mlp(h, w.view(np.uint16), np.random.default_rng(0).uniform(0, 1, 16))
    np.testing.assert_array_equal(y, [0.25, 0.5, 0.75])


def test_half_to_double_exact():
    lib = oracle.lib()
    for bits in [0x0000, 0x0001, 0x03FF, 0x0400, 0x3C00, 0x3555, 0x7BFF, 0x8001, 0xBC00, 0xC000]:
        exp = float(np.array([bits], np.uint16).view(np.float16)[0])
        assert lib.oracle_half_to_double(bits) == exp
