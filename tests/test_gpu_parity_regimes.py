"""GPU parity outside the seeded numeric regime (VERDICT r1 "parity partial").

The default synthetic weights (nn.Linear init, b3 += 0.5) keep the decoder's
output in about [0.03, 0.7] and its hidden pre-activations small.  These tests
drive the fused tensor-core path (NDGI_MODE_FAST) through the regimes the
method also has, element by element against the fp64 oracle:

* "stress" weights (ndgi_synth MLP_SCALES): hidden pre-activations up to
  |z| ~ 10 -- the polynomial GELU's clamped tail and large-magnitude f16
  operands -- and ~10 % of the outputs below 0 / above 1, so the RGBA8 clamp of
  R12 ("quantized into an 8-bit 4-channel format") is hit on both sides;
* a Theta produced by the GPU trainer and exported (R30), decoded in FAST mode;
* BC7 reserved mode 8 (R9) through the B200 texture unit;
* config 3's exact VT bench launch (16,384-tile scene, n = 512 random ids,
  decode_tiles RGBA8), checked per slot;
* a border wider than half the core (2B > C - 2), where a core texel has both
  mirror images (R3).

Bars as in test_gpu_decode.py: FAST max-abs <= 2e-2 / mean-abs <= 2e-3 on
RGBA32F, RGBA8 = the oracle's quantiser of the kernel's own y and within one
level of the oracle's y, REF_FP32 <= 1e-5.
"""
import os

import numpy as np
import pytest

import ndgi_synth as S
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2604_12625_b200 as ndgi  # noqa: E402

from test_gpu_decode import FAST_MAX, FAST_MEAN, REF_MAX, _err, _load, gpu_full, gpu_tiles  # noqa: E402

NTHR = max(1, len(os.sched_getaffinity(0)))


# The RGBA8 level bar implied by the FAST RGB bar (north_star max-abs 2e-2):
# |q_kernel - q_oracle| <= 255 * 2e-2 + 1 rounding boundary.  The default-weight
# tests (test_gpu_decode.py) keep SURVEY's stricter 1 level, which holds there;
# trained weights with outputs far outside [0, 1] reach ~1e-2 (R32).
RGBA8_LEVELS_FAST = int(255 * FAST_MAX) + 1


def _check_rgba8(q8, y32, exp, levels=1):
    """RGBA8 == the oracle's fp32 quantiser of the kernel's own y (same precision,
    R12), and within `levels` of the oracle's fp64 y; clamped texels (oracle y
    outside [0, 1] by more than the FAST tolerance) are exactly 0 / 255."""
    np.testing.assert_array_equal(q8, oracle.quantize_rgba8(np.ascontiguousarray(y32)))
    qe = oracle.quantize_rgba8(np.ascontiguousarray(exp))
    d = np.abs(q8[..., :3].astype(int) - qe[..., :3].astype(int))
    assert d.max() <= levels, d.max()
    lo, hi = exp < -FAST_MAX, exp > 1 + FAST_MAX
    assert (q8[..., :3][lo] == 0).all() and (q8[..., :3][hi] == 255).all()


STRESS_CASES = {
    "M": S.layout(1, 2, 2, "M", uvt_depth=4, line_t=4),
    "M-tanh": S.layout(1, 2, 2, "M", uvt_depth=4, line_t=4, gelu="tanh"),
    "H": S.layout(1, 2, 2, "H", uvt_depth=4, line_t=4),            # windowed F_uvt
    "L-u8": S.layout(1, 2, 2, "L", uvt_depth=4, line_t=4, fmt_uv="u8", fmt_uvt="u8"),
    "M64": S.layout(1, 2, 2, "M64", uvt_depth=4, line_t=4),
}


@pytest.mark.parametrize("name", list(STRESS_CASES))
def test_stress_weights_fast_parity(name):
    lay = STRESS_CASES[name]
    th = S.make_theta(lay, 61, "smooth", mlp="stress")
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    C, B = lay["core"], lay["border"]
    for t in (0.3, 0.875):
        exp = M.decode_full(t, NTHR)[0]
        # the regime is really reached: outputs leave [0, 1] on both sides
        assert (exp < 0).mean() > 0.005 and (exp > 1).mean() > 0.005, name
        y32 = gpu_full(ctx, t, "rgba32f", "fast")[0, 0]
        mx, mean = _err(y32, exp)
        print(f"stress {name} t={t}: max {mx:.3e} mean {mean:.3e}")
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (name, t, mx, mean)
        # FULL8 (decode_full RGBA8)
        q8 = gpu_full(ctx, t, "rgba8", "fast")[0, 0]
        _check_rgba8(q8, y32, exp)
        # REF_FP32 stays within 1e-5 in this regime too
        ref = gpu_full(ctx, t, "rgba32f", "ref_fp32")[0, 0]
        assert _err(ref, exp)[0] <= REF_MAX
    # TILES8 (decode_tiles RGBA8, mirrored border): against the oracle's padded tiles
    ids, slots, t = [3, 0, 2, 1], [1, 3, 0, 2], 0.55
    q = gpu_tiles(ctx, ids, t, "rgba8", slots=slots)
    y = gpu_tiles(ctx, ids, t, "rgba32f", slots=slots)
    exp = M.decode_tiles(ids, t, NTHR)
    for r, s in enumerate(slots):
        mx, mean = _err(y[s], exp[r])
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (name, r, mx, mean)
        _check_rgba8(q[s], y[s], exp[r])


def test_trained_exported_theta_fast_parity():
    """A Theta the GPU trainer produced (full step R28, a few hundred Adam steps
    at a large learning rate) and exported (R30: u8 PTQ + BC7 mode 6 + f16
    MLP), loaded into a FAST layout and decoded with the tensor-core path."""
    lay = S.layout(1, 2, 2, "M", uvt_depth=4, line_t=4)
    th0 = S.make_theta(lay, 9, "smooth")
    ctx = _load(lay, th0)
    P = ndgi.train_full_params(lay)
    h = lay["hidden"]
    pm = 16 * h + h + h * h + h + 3 * h + 3
    rng = np.random.default_rng(4)
    init = np.concatenate([rng.normal(0, 0.6, (4, pm)), rng.uniform(0.05, 0.95, (4, P - pm))], 1).astype(np.float32)
    tr = ndgi.Trainer(ctx, full_init=torch.from_numpy(init).cuda())
    tiles = [0, 1, 2, 3]
    Sn = 4096
    smp, tgt = S.train_batch(tiles, Sn, 12)
    tgt = (tgt - 0.5) * 1.6 + 0.5                      # targets in about [-0.14, 1.14]: outputs leave [0, 1]
    ids = torch.tensor(tiles, dtype=torch.int32, device="cuda")
    smp_t, tgt_t = torch.from_numpy(smp).cuda(), torch.from_numpy(tgt.astype(np.float32)).cuda()
    g = torch.Generator(device="cuda").manual_seed(3)
    lo = torch.zeros(4, device="cuda")
    first = None
    for it in range(300):
        noise = torch.rand((4, Sn, 12), device="cuda", generator=g) - 0.5
        tr.step(ids, smp_t, tgt_t, lr=1e-2, loss=lo, noise=noise)
        if it == 0:
            first = lo.cpu().numpy().copy()
    assert (lo.cpu().numpy() < first).all()
    out = tr.export_full()
    torch.cuda.synchronize()
    th = {k: v.cpu().numpy() for k, v in out.items()}
    th["mlp"] = th["mlp"].view(np.uint16)
    w = th["mlp"].view(np.float16).astype(np.float64)
    assert np.abs(w).max() > 1.0                       # trained weights, not the init scale
    M = oracle.Model(lay, th)
    ctx2 = ndgi.ndgi_load(lay, out, 0)
    for t in (0.2, 13 / 24):
        exp = M.decode_full(t, NTHR)[0]
        y32 = gpu_full(ctx2, t, "rgba32f", "fast")[0, 0]
        mx, mean = _err(y32, exp)
        print(f"trained t={t}: max {mx:.3e} mean {mean:.3e}, y in [{exp.min():.2f}, {exp.max():.2f}]")
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (t, mx, mean)
        assert (exp < 0).mean() > 0.005 and (exp > 1).mean() > 0.005
        _check_rgba8(gpu_full(ctx2, t, "rgba8", "fast")[0, 0], y32, exp, RGBA8_LEVELS_FAST)
    tr.close()


def test_bc7_mode8_texture_unit():
    """R9 against the hardware: reserved mode-8 blocks (byte 0 = 0) decode to
    (0, 0, 0, 0) in the B200 texture unit, in the kernel's decoder and in the
    oracle (Pillow differs: A = 255, so it is excluded from the Pillow pin)."""
    w = h = 64
    n = (w // 4) * (h // 4)
    words = S.splitmix64(np.arange(2 * n, dtype=np.uint64) + np.uint64(1234)).reshape(n, 2)
    blocks = S.bc7_random_blocks(words, np.full(n, 8))
    assert (blocks[:, 0] == 0).all()
    exp = oracle.bc7_decode_image(blocks, w, h)
    assert (exp == 0).all()
    hw = torch.zeros((h, w, 4), dtype=torch.uint8, device="cuda")
    ndgi.ndgi_debug_bc7_decode_hw(torch.from_numpy(blocks.copy()).cuda(), w, h, hw)
    sw = torch.zeros((h, w, 4), dtype=torch.uint8, device="cuda")
    ndgi.ndgi_debug_bc7_decode(torch.from_numpy(blocks.copy()).cuda(), w, h, sw)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hw.cpu().numpy(), exp)
    np.testing.assert_array_equal(sw.cpu().numpy(), exp)


_C3 = {}


def _c3():
    if not _C3:
        lay, seed = S.config("c3")
        th = S.make_theta(lay, seed)
        _C3.update(lay=lay, seed=seed, th=th, ctx=_load(lay, th))
    return _C3["lay"], _C3["seed"], _C3["th"], _C3["ctx"]


def _tile_oracle_padded(lay, seed, ids, t):
    lay1 = S.layout(1, len(ids), 1, "M")
    return oracle.Model(lay1, S.make_theta(lay1, seed, tiles=list(ids))).decode_tiles(list(range(len(ids))), t, NTHR)


def test_c3_vt_bench_launch_per_slot():
    """bench.py's VT leg exactly: config 3's 16,384-tile scene, the first frame's
    n = 512 random ids and t, slots 0..n-1, decode_tiles RGBA8 (TILES8 kernel,
    whole-tile units).  Every slot: 64 sampled padded texels (border included)
    against the oracle's RGBA8 within one level; 6 whole slots exactly
    quantiser-equal to the kernel's own RGBA32F and within one level."""
    lay, seed, th, ctx = _c3()
    n = 512
    ids, t = S.vt_batches(lay["num_tiles"], n, 1, seed)[0]
    q = gpu_tiles(ctx, ids, t, "rgba8")
    assert ndgi.ndgi_device_error(ctx, reset=True) == 0
    P, B = 136, 4
    rng = np.random.default_rng(5)
    for s in range(n):
        k = int(ids[s])
        Mk = oracle.Model(S.layout(1, 1, 1, "M"), {key: v[k:k + 1] for key, v in th.items()})
        xs = rng.integers(0, P, 64)
        ys = rng.integers(0, P, 64)
        for x, y in zip(xs, ys):
            e = oracle.quantize_rgba8(Mk.texel(0, int(x), int(y), t).reshape(1, 3))[0]
            assert np.abs(q[s, y, x].astype(int) - e.astype(int)).max() <= 1, (s, k, x, y)
    whole = [0, 1, 100, 255, 256, 511]
    y32 = gpu_tiles(ctx, ids, t, "rgba32f")
    exp = _tile_oracle_padded(lay, seed, [int(ids[s]) for s in whole], t)
    for r, s in enumerate(whole):
        mx, mean = _err(y32[s], exp[r])
        assert mx <= FAST_MAX and mean <= FAST_MEAN
        np.testing.assert_array_equal(q[s], oracle.quantize_rgba8(np.ascontiguousarray(y32[s])))
        assert np.abs(q[s][..., :3].astype(int) - oracle.quantize_rgba8(exp[r])[..., :3].astype(int)).max() <= 1


@pytest.mark.parametrize("border", [63, 64, 100])
def test_wide_border_both_mirrors(border):
    """2B > C - 2: core texels near the middle have both mirror images in the
    padded tile (R3).  FAST decode_tiles (RGBA8 and RGBA32F) must
    equal F.pad(reflect) of its own core, and the oracle within the FAST bars."""
    lay = S.layout(1, 2, 1, "M", border=border, uvt_depth=4, line_t=4)
    th = S.make_theta(lay, 5)
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    C, B = 128, border
    ids = [1, 0]
    for fmt in ("rgba8", "rgba32f"):
        got = gpu_tiles(ctx, ids, 0.4, fmt)
        for r in range(2):
            core = got[r, B:B + C, B:B + C]
            pad = np.asarray(torch.nn.functional.pad(torch.from_numpy(np.ascontiguousarray(core.astype(np.float32)))
                                                     .permute(2, 0, 1)[None], (B, B, B, B), mode="reflect")[0]
                             .permute(1, 2, 0).numpy()).astype(core.dtype)
            np.testing.assert_array_equal(got[r], pad)
    y = gpu_tiles(ctx, ids, 0.4, "rgba32f")
    exp = M.decode_tiles(ids, 0.4, NTHR)
    for r in range(2):
        mx, mean = _err(y[r], exp[r])
        assert mx <= FAST_MAX and mean <= FAST_MEAN


RING_CASES = {
    # the F_uvt ring (R3 > 32) off the H profile's power-of-two size
    "R3=48-bc7": S.layout(1, 2, 1, "M", uvt_res=48, uvt_depth=4, line_t=4),
    "R3=40-u8": S.layout(1, 2, 1, "M", uvt_res=40, uvt_depth=4, line_t=4, fmt_uv="u8", fmt_uvt="u8"),
    "R3=36-f16": S.layout(1, 2, 1, "M", uvt_res=36, uvt_depth=4, line_t=4, fmt_uv="f16", fmt_uvt="f16",
                          fmt_line="f16"),
    "R3=33-u8": S.layout(1, 2, 1, "M", uvt_res=33, uvt_depth=3, line_t=4, fmt_uv="u8", fmt_uvt="u8"),
    "R3=56-bc1": S.layout(1, 2, 1, "M", uvt_res=56, uvt_depth=4, line_t=8, fmt_uv="bc1", fmt_uvt="bc1",
                          fmt_line="bc5"),
}


@pytest.mark.parametrize("name", list(RING_CASES))
def test_uvt_ring_sizes(name):
    """F_uvt rings for R3 in (32, 64] that are not powers of two, including
    dense maps whose R3 is not a multiple of 4 (ring staging of partial block
    columns): decode_full and decode_tiles with 4-row strips vs the oracle."""
    lay = RING_CASES[name]
    th = S.make_theta(lay, 23, "mixed")
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    for t in (0.2, 0.95):
        y = gpu_full(ctx, t, "rgba32f", "fast")[0, 0]
        mx, mean = _err(y, M.decode_full(t, NTHR)[0])
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (name, t, mx, mean)
    got = gpu_tiles(ctx, [1], 0.61, "rgba32f")      # n = 1: 4-row strips, ring restaged per strip
    mx, mean = _err(got, M.decode_tiles([1], 0.61, NTHR))
    assert mx <= FAST_MAX and mean <= FAST_MEAN, (name, mx, mean)


EDGE_CASES = {
    "C256-R3=64": S.layout(1, 1, 1, "H", core=256, uv_res=256, uvt_depth=3, line_t=4),   # whole 32 KB slice
    "D1-T1": S.layout(1, 2, 1, "M", uvt_depth=1, line_t=1),                             # single slice / row
    "R3=4-U=1": S.layout(1, 2, 1, "M", uvt_res=4, line_res=1, uvt_depth=2, line_t=3),   # smallest maps
    "M64-C256": S.layout(1, 1, 1, "M64", core=256, uv_res=256, uvt_depth=2, line_t=2),
}


@pytest.mark.parametrize("name", list(EDGE_CASES))
def test_fast_layout_edges(name):
    """FAST-mode layouts at the edges of what the fused kernel takes: C = 256
    with the whole R3 = 64 slice in smem, a single F_uvt slice and line row
    (k0 = k1, r0 = r1), the smallest maps (R3 = 4, U = 1), h = 64 with C = 256 —
    decode_full at t = 0, 0.5, 1 and decode_tiles against the oracle."""
    lay = EDGE_CASES[name]
    th = S.make_theta(lay, 31, "mixed")
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    for t in (0.0, 0.5, 1.0):
        y = gpu_full(ctx, t, "rgba32f", "fast")[0, 0]
        mx, mean = _err(y, M.decode_full(t, NTHR)[0])
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (name, t, mx, mean)
    ids = list(range(lay["num_tiles"]))
    got = gpu_tiles(ctx, ids, 0.7, "rgba32f")
    mx, mean = _err(got, M.decode_tiles(ids, 0.7, NTHR))
    assert mx <= FAST_MAX and mean <= FAST_MEAN, (name, mx, mean)
