"""Pins of the oracle's shading side (readings R21-R25):
mean interpolation against numpy.interp, the restore against the SPEC's worked
examples and a numpy round trip of the preprocessing it inverts, and the
page-cache sampler against scipy's bilinear map_coordinates, closed forms
(linear ramps are reproduced exactly by bilinear filtering) and the mirrored
border built by numpy.pad(mode="reflect")."""
import numpy as np
import pytest
from scipy import ndimage

import oracle


# ------------------------------------------------------------------ R22 means
def test_mean_at_matches_numpy_interp():
    rng = np.random.default_rng(7)
    times = np.sort(rng.uniform(0, 1, 9))
    times[0], times[-1] = 0.0, 1.0
    means = rng.uniform(0.1, 5.0, (9, 3))
    for t in np.concatenate([times, rng.uniform(0, 1, 50)]):
        got = oracle.mean_at(times, means, t)
        exp = np.array([np.interp(t, times, means[:, c]) for c in range(3)])
        np.testing.assert_allclose(got, exp, rtol=1e-14, atol=1e-14)


def test_mean_at_frame_times_and_range():
    times = np.array([0.0, 0.5, 1.0])
    means = np.array([[1.0, 1.0, 1.0], [2.0, 3.0, 4.0], [4.0, 3.0, 2.0]])
    np.testing.assert_array_equal(oracle.mean_at(times, means, 0.5), means[1])
    # SPEC postprocess example: mu interpolated midway between 2.0 and 4.0 -> 3.0
    np.testing.assert_allclose(oracle.mean_at(times, means, 0.75)[0], 3.0, rtol=0, atol=1e-15)
    for bad in (-1e-9, 1.0 + 1e-9, float("nan")):
        with pytest.raises(ValueError):
            oracle.mean_at(times, means, bad)
    assert np.array_equal(oracle.mean_at(np.array([0.3]), np.array([[2.0, 3.0, 4.0]]), 0.3), [2.0, 3.0, 4.0])


# ------------------------------------------------------------------ R21/R23 restore
def test_restore_examples_and_round_trip():
    assert oracle.restore(1.0, 2.2, 1.0) == 1.0           # SPEC: value 1.0 at frame time, mu = 1 -> 1.0
    assert oracle.restore(0.0, 2.2, 5.0) == 0.0
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 40, 1000)                          # linear HDR texels
    mu = rng.uniform(0.5, 20, 1000)
    g = 2.2
    pre = (x / mu) ** (1.0 / g)                           # the preprocessing, numpy
    back = np.array([oracle.restore(p, g, m) for p, m in zip(pre, mu)])
    np.testing.assert_allclose(back, x, rtol=1e-12)


# ------------------------------------------------------------------ R24/R25 sampler
def _cache(slots, C, B, rng):
    P = C + 2 * B
    return rng.integers(0, 256, (slots, P, P, 4), dtype=np.uint8)


def test_texel_centre_samples_are_the_texels():
    rng = np.random.default_rng(11)
    C, B, tx, ty = 8, 2, 3, 2
    cache = _cache(tx * ty, C, B, rng)
    pt = np.stack([np.arange(tx * ty)[::-1], np.zeros(tx * ty, int)], 1).astype(np.int32)   # reversed slots
    W, H = tx * C, ty * C
    ii, jj = np.meshgrid(np.arange(W), np.arange(H))
    uv = np.stack([(ii.ravel() + 0.5) / W, (jj.ravel() + 0.5) / H], 1)
    mu = np.array([[1.5, 2.0, 0.5]])
    got, ok = oracle.sample_lighting(cache, pt, C, B, tx, ty, np.zeros(len(uv), int), uv, 0, 2.2, mu)
    assert ok.all()
    tile = (jj.ravel() // C) * tx + ii.ravel() // C
    slot = pt[tile, 0]
    q = cache[slot, jj.ravel() % C + B, ii.ravel() % C + B, :3] / 255.0
    np.testing.assert_allclose(got, q ** 2.2 * mu[0], rtol=1e-13, atol=1e-15)


def test_bilinear_against_scipy_map_coordinates():
    rng = np.random.default_rng(5)
    C, B = 16, 4
    cache = _cache(1, C, B, rng)
    pt = np.array([[0, 3]], np.int32)
    uv = rng.uniform(0, 1, (400, 2))
    got, ok = oracle.sample_lighting(cache, pt, C, B, 1, 1, np.zeros(400, int), uv, 3, 1.0, np.ones((1, 3)))
    assert ok.all()
    # padded-slot coordinates of the samples; scipy's order-1 spline = bilinear
    xs = uv[:, 0] * C - 0.5 + B
    ys = uv[:, 1] * C - 0.5 + B
    for c in range(3):
        exp = ndimage.map_coordinates(cache[0, :, :, c].astype(np.float64) / 255.0, [ys, xs], order=1, mode="nearest")
        np.testing.assert_allclose(got[:, c], exp, rtol=0, atol=1e-12)


def test_linear_ramp_is_reproduced_exactly():
    # bilinear filtering reproduces an affine field exactly (closed form)
    C, B = 32, 4
    P = C + 2 * B
    y, x = np.mgrid[0:P, 0:P]
    cache = np.zeros((1, P, P, 4), np.uint8)
    cache[0, :, :, 0] = 2 * x + 3 * y          # <= 2*39 + 3*39 = 195
    cache[0, :, :, 1] = 5 * x
    cache[0, :, :, 2] = 6 * y
    rng = np.random.default_rng(2)
    uv = rng.uniform(0, 1, (300, 2))
    got, _ = oracle.sample_lighting(cache, np.array([[0, 0]], np.int32), C, B, 1, 1, np.zeros(300, int), uv, 0, 1.0,
                                    np.ones((1, 3)))
    X = uv[:, 0] * C - 0.5 + B
    Y = uv[:, 1] * C - 0.5 + B
    np.testing.assert_allclose(got[:, 0], (2 * X + 3 * Y) / 255, atol=1e-12)
    np.testing.assert_allclose(got[:, 1], 5 * X / 255, atol=1e-12)
    np.testing.assert_allclose(got[:, 2], 6 * Y / 255, atol=1e-12)


def test_tile_edges_use_the_mirrored_border():
    # two tiles side by side, borders = numpy reflect padding of each core
    # (R3); at the shared edge each side filters with its own border
    rng = np.random.default_rng(9)
    C, B = 8, 4
    cores = rng.integers(0, 256, (2, C, C, 3)).astype(np.uint8)
    cache = np.zeros((2, C + 2 * B, C + 2 * B, 4), np.uint8)
    for k in range(2):
        cache[k, :, :, :3] = np.pad(cores[k], ((B, B), (B, B), (0, 0)), mode="reflect")
    pt = np.array([[0, 0], [1, 0]], np.int32)
    W = 2 * C
    j = 3
    v = (j + 0.5) / C
    eps = 1e-9
    # just left of the edge: tile 0, local x = C - 0.5 - eps*W -> taps C-1 and C (= core C-2)
    # with weight 0.5 - eps*W on the border tap
    uv = np.array([[0.5 - eps, v], [0.5, v], [0.0, v], [1.0, v], [-0.3, v], [1.7, v]])
    got, ok = oracle.sample_lighting(cache, pt, C, B, 2, 1, np.zeros(len(uv), int), uv, 0, 1.0, np.ones((1, 3)))
    assert ok.all()
    c0 = cores[0, j].astype(np.float64) / 255
    c1 = cores[1, j].astype(np.float64) / 255
    fx = 0.5 - eps * W                                   # weight of tap x = C (the border) near the edge
    np.testing.assert_allclose(got[0], (1 - fx) * c0[C - 1] + fx * c0[C - 2], atol=1e-6)
    # exactly on the edge: tile 1 (floor), local x = -0.5 -> taps -1 (= core 1) and 0, half each
    np.testing.assert_allclose(got[1], 0.5 * c1[1] + 0.5 * c1[0], atol=1e-12)
    np.testing.assert_allclose(got[2], 0.5 * c0[1] + 0.5 * c0[0], atol=1e-12)           # u = 0
    np.testing.assert_allclose(got[3], 0.5 * c1[C - 1] + 0.5 * c1[C - 2], atol=1e-12)   # u = 1
    np.testing.assert_array_equal(got[4], got[2])                                       # clamp
    np.testing.assert_array_equal(got[5], got[3])


def test_residency_and_indirection():
    rng = np.random.default_rng(4)
    C, B, T = 8, 2, 4
    cache = _cache(T, C, B, rng)
    uv = rng.uniform(0, 1, (200, 2))
    at = np.zeros(200, int)
    ident = np.stack([np.arange(T), np.full(T, 7)], 1).astype(np.int32)
    a, ok_a = oracle.sample_lighting(cache, ident, C, B, 2, 2, at, uv, 7, 2.2, np.ones((1, 3)))
    perm = np.array([2, 0, 3, 1])
    cache_p = np.empty_like(cache)
    cache_p[perm] = cache                                    # tile k now lives in slot perm[k]
    pt_p = np.stack([perm, np.full(T, 7)], 1).astype(np.int32)
    b, ok_b = oracle.sample_lighting(cache_p, pt_p, C, B, 2, 2, at, uv, 7, 2.2, np.ones((1, 3)))
    assert ok_a.all() and ok_b.all()
    np.testing.assert_array_equal(a, b)
    # wrong bucket / absent tile -> not resident
    _, ok = oracle.sample_lighting(cache, ident, C, B, 2, 2, at, uv, 6, 2.2, np.ones((1, 3)))
    assert not ok.any()
    absent = ident.copy()
    absent[3, 0] = -1
    _, ok = oracle.sample_lighting(cache, absent, C, B, 2, 2, at, uv, 7, 2.2, np.ones((1, 3)))
    owner = (np.minimum((uv[:, 1] * 2).astype(int), 1)) * 2 + np.minimum((uv[:, 0] * 2).astype(int), 1)
    np.testing.assert_array_equal(ok, owner != 3)


def test_atlas_addressing():
    rng = np.random.default_rng(8)
    C, B = 8, 2
    cache = _cache(4, C, B, rng)                 # 2 atlases x (1 x 2) tiles
    pt = np.stack([np.arange(4), np.zeros(4, int)], 1).astype(np.int32)
    uv = np.array([[0.25, 0.5], [0.75, 0.5]])
    mu = np.array([[1.0, 1.0, 1.0], [2.0, 2.0, 2.0]])
    a0, _ = oracle.sample_lighting(cache, pt, C, B, 2, 1, np.array([0, 0]), uv, 0, 1.0, mu)
    a1, _ = oracle.sample_lighting(cache, pt, C, B, 2, 1, np.array([1, 1]), uv, 0, 1.0, mu)
    c = C // 2 + B   # texel (C/2 - 0.5) -> lerp of C/2-1 and C/2
    for s, (got, slot) in enumerate([(a0[0], 0), (a0[1], 1), (a1[0], 2), (a1[1], 3)]):
        q = 0.5 * (cache[slot, B + C // 2, c - 1, :3].astype(float) + cache[slot, B + C // 2, c, :3]) / 255
        q = 0.5 * q + 0.5 * 0.5 * (cache[slot, B + C // 2 - 1, c - 1, :3].astype(float) +
                                   cache[slot, B + C // 2 - 1, c, :3]) / 255
        np.testing.assert_allclose(got, q * (2.0 if slot >= 2 else 1.0), atol=1e-12)
