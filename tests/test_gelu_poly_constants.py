"""Host check of the FMA-pipe GELU polynomial in csrc/ndgi_common.cuh
(`gelu_poly_f16x2`): the f16 coefficients baked into the
kernel source, evaluated in fp64, approximate tanh(h (1 + c h^2)) on the clamp
range [0, 2.5] and, through the clamp hc = min(h, 2.5), on the whole half-line
(the function is odd), within the error the design states.  c = 0.044715 / (2/pi)
(the tanh-GELU of P:234 with sqrt(2/pi) folded into h)."""
import math
import os
import re

import numpy as np
import pytest

SRC = os.path.join(os.path.dirname(__file__), "..", "paper_2604_12625_b200", "csrc", "ndgi_common.cuh")
C = 0.044715 / (2.0 / math.pi)


def _coeffs(deg4: bool):
    src = open(SRC).read()
    body = src[src.index("gelu_poly_f16x2(uint32_t h)"):]
    body = body[:body.index("return g;")]
    a, b = body.split("#if NDGI_POLY_DEG4")[1].split("#else")
    b = b.split("#endif")[0]
    hexes = re.findall(r"0x([0-9A-Fa-f]{4})\1u", a if deg4 else b)
    vals = [float(np.array([int(x, 16)], np.uint16).view(np.float16)[0]) for x in hexes]
    # first FMA: s * k_hi + k_next; then q = q * s + k for each remaining constant
    return vals


@pytest.mark.parametrize("deg4,bound", [(True, 1.0e-3), (False, 3.0e-3)])
def test_poly_fit_error(deg4, bound):
    k = _coeffs(deg4)
    assert len(k) == (5 if deg4 else 6)
    h = np.linspace(0.0, 8.0, 80001)
    hc = np.minimum(h, 2.5)
    s = hc * hc
    q = k[0] * s + k[1]
    for kk in k[2:]:
        q = q * s + kk
    err = np.abs(hc * q - np.tanh(h * (1 + C * h * h)))
    assert err.max() <= bound, err.max()


def test_clamp_constant_is_f16_2_5():
    assert "0x41004100u" in open(SRC).read() and "0xC100C100u" in open(SRC).read()
    assert float(np.array([0x4100], np.uint16).view(np.float16)[0]) == 2.5
    assert float(np.array([0xC100], np.uint16).view(np.float16)[0]) == -2.5
