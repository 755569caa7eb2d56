"""GPU parity of libndgi.so against the CPU oracle (called through the C ABI).

Bars (BASELINE.json north_star):
* BC7 decode: bit-exact (device decoder vs oracle; vs the B200 texture unit);
* NDGI_MODE_REF_FP32: max-abs <= 1e-5 on RGBA32F vs the fp64 oracle;
* NDGI_MODE_FAST (tcgen05, f16 operands): max-abs <= 2e-2, mean-abs <= 2e-3;
* RGBA8: the kernel's quantisation of its own fp32 y equals RN-even(clamp(y)*255)
  computed by the oracle in fp32 (same precision), and |dq| <= 1 vs the oracle's y.
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

NTHR = max(1, len(os.sched_getaffinity(0)))
FAST_MAX, FAST_MEAN, REF_MAX = 2e-2, 2e-3, 1e-5


def _load(lay, th):
    return ndgi.ndgi_load(lay, ndgi.upload_theta(th), 0)


def gpu_full(ctx, ts, fmt="rgba32f", mode="fast"):
    ts = [ts] if np.isscalar(ts) else list(ts)
    L = ctx.lay
    C = L["core"]
    shape = (len(ts), L["atlases"], L["tiles_y"] * C, L["tiles_x"] * C)
    if fmt == "rgba8":
        out = torch.zeros(shape + (4,), dtype=torch.uint8, device="cuda")
    elif fmt == "rgba16f":
        out = torch.zeros(shape + (4,), dtype=torch.float16, device="cuda")
    else:
        out = torch.zeros(shape + (4,), dtype=torch.float32, device="cuda")
    if len(ts) == 1:
        ndgi.ndgi_decode_full(ctx, ts[0], out, fmt, mode)
    else:
        ndgi.ndgi_decode_full_batch(ctx, ts, out, fmt, mode)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def gpu_tiles(ctx, ids, t, fmt="rgba32f", mode="fast", slots=None, num_slots=None):
    P = ctx.padded
    n = len(ids)
    num_slots = num_slots or n
    dt = {"rgba8": torch.uint8, "rgba16f": torch.float16, "rgba32f": torch.float32}[fmt]
    out = torch.zeros((num_slots, P, P, 4), dtype=dt, device="cuda")
    ids_t = torch.tensor(np.asarray(ids, np.int64), dtype=torch.int32, device="cuda")
    sl_t = None if slots is None else torch.tensor(np.asarray(slots, np.int64), dtype=torch.int32, device="cuda")
    ndgi.ndgi_decode_tiles(ctx, ids_t, sl_t, n, num_slots, t, out, fmt, mode)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _err(got, exp):
    d = np.abs(got[..., :3].astype(np.float64) - exp)
    return float(d.max()), float(d.mean())


# ------------------------------------------------------------------ BC7
def _mixed_blocks(n, seed, with_mode8=True):
    words = S.splitmix64(np.arange(3 * n, dtype=np.uint64) + np.uint64(seed)).reshape(n, 3)
    modes = (words[:, 2] % np.uint64(9 if with_mode8 else 8)).astype(np.int64)
    return S.bc7_random_blocks(words[:, :2], modes)


@pytest.mark.parametrize("payload", ["mixed", "smooth", "mode6"])
def test_bc7_device_decoder_bit_exact(payload):
    w = h = 512
    n = (w // 4) * (h // 4)
    if payload == "mixed":
        blocks = _mixed_blocks(n, 17)
    elif payload == "mode6":
        blocks = _mixed_blocks(n, 5, False)
        words = S.splitmix64(np.arange(2 * n, dtype=np.uint64) + np.uint64(99)).reshape(n, 2)
        blocks = S.bc7_random_blocks(words, np.full(n, 6))
    else:
        lay = S.layout(1, 4, 4, "M")
        blocks = S.make_theta(lay, 3)["uv"].reshape(n, 16)
    exp = oracle.bc7_decode_image(blocks, w, h)
    dev_blocks = torch.from_numpy(blocks.copy()).cuda()
    out = torch.zeros((h, w, 4), dtype=torch.uint8, device="cuda")
    ndgi.ndgi_debug_bc7_decode(dev_blocks, w, h, out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), exp)


def test_bc7_texture_unit_agrees_with_oracle():
    """The B200's own BC7 decoder (texture unit) as an independent reference."""
    w = h = 256
    n = (w // 4) * (h // 4)
    blocks = _mixed_blocks(n, 23, with_mode8=False)
    exp = oracle.bc7_decode_image(blocks, w, h)
    out = torch.zeros((h, w, 4), dtype=torch.uint8, device="cuda")
    ndgi.ndgi_debug_bc7_decode_hw(torch.from_numpy(blocks.copy()).cuda(), w, h, out)
    np.testing.assert_array_equal(out.cpu().numpy(), exp)


# ------------------------------------------------------------------ reference mode
@pytest.mark.parametrize("gelu", ["erf", "tanh"])
def test_ref_fp32_full_c1(gelu):
    lay, seed = S.config("c1")
    lay = dict(lay, gelu=gelu)
    th = S.make_theta(lay, seed)
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    for t in (0.3, 0.375, 0.0, 1.0):
        got = gpu_full(ctx, t, "rgba32f", "ref_fp32")[0]
        exp = M.decode_full(t, NTHR)
        mx, mean = _err(got, exp)
        assert mx <= REF_MAX, (t, mx, mean)
        assert (got[..., 3] == 1.0).all()


def test_ref_fp32_tiles_slots_and_small_cores():
    # ragged geometry the fast path does not take: C=12, R_uv=8 (bilinear F_uv), h=8, eval-clamp border
    for lay in (S.layout(1, 3, 1, "M", core=12, border=3, uv_res=8, uvt_res=8, uvt_depth=3, line_res=7, line_t=5, hidden=8),
                S.layout(1, 2, 1, "M", core=8, border=4, uvt_res=4, uvt_depth=2, line_res=4, line_t=2, hidden=4,
                         border_mode="eval_clamp", fmt_uv="f16", fmt_uvt="u8", fmt_line="f16")):
        th = S.make_theta(lay, 7, "mixed")
        M = oracle.Model(lay, th)
        ctx = _load(lay, th)
        ids = [1, 0, 2][:lay["num_tiles"]] + [0]
        slots = list(range(len(ids)))[::-1]
        got = gpu_tiles(ctx, ids, 0.61, "rgba32f", "ref_fp32", slots=slots, num_slots=len(ids) + 1)
        exp = M.decode_tiles(ids, 0.61)
        for r, s in enumerate(slots):
            mx, _ = _err(got[s], exp[r])
            assert mx <= REF_MAX, (lay["core"], r, mx)


# ------------------------------------------------------------------ fast (tensor-core) mode
FAST_CASES = {
    "c1-bc7": (S.config("c1")[0], "smooth"),
    "c1-bc7-mixed": (S.config("c1")[0], "mixed"),
    "u8": (S.layout(1, 2, 1, "M", uvt_depth=5, line_t=7, fmt_uv="u8", fmt_uvt="u8"), "smooth"),
    "f16": (S.layout(1, 2, 1, "M", uvt_depth=5, line_t=7, fmt_uv="f16", fmt_uvt="f16", fmt_line="f16"), "smooth"),
    "M64": (S.layout(1, 2, 1, "M64", uvt_depth=4, line_t=4), "smooth"),
    "L-tanh": (S.layout(1, 2, 1, "L", gelu="tanh"), "smooth"),
    "H": (S.layout(1, 1, 2, "H"), "mixed"),          # R3 = 64: windowed F_uvt (BC7 windows)
    "H-u8": (S.layout(1, 2, 1, "H", fmt_uv="u8", fmt_uvt="u8"), "smooth"),
    "H-f16": (S.layout(1, 2, 1, "H", fmt_uv="f16", fmt_uvt="f16", fmt_line="f16"), "smooth"),
    "C256": (S.layout(1, 1, 1, "M", core=256, uv_res=256), "smooth"),
    # R29: the other DXTC formats (config 5's BC-format axis)
    "bc3-bc5": (S.layout(1, 2, 1, "M", uvt_depth=4, line_t=8, fmt_uv="bc3", fmt_uvt="bc3", fmt_line="bc5"), "smooth"),
    "bc1-bc5-mixed": (S.layout(1, 2, 1, "M", uvt_depth=4, line_t=8, fmt_uv="bc1", fmt_uvt="bc1", fmt_line="bc5"),
                      "mixed"),
    "H-bc3": (S.layout(1, 1, 2, "H", fmt_uv="bc3", fmt_uvt="bc3", fmt_line="bc5"), "mixed"),   # windowed F_uvt
    "H-bc1": (S.layout(1, 1, 2, "H", fmt_uv="bc1", fmt_uvt="bc1", fmt_line="bc5"), "mixed"),   # 3-colour blocks too
}


@pytest.mark.parametrize("name", list(FAST_CASES))
def test_fast_full_parity(name):
    lay, payload = FAST_CASES[name]
    th = S.make_theta(lay, 41, payload)
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    for t in (0.3, 1.0):
        got = gpu_full(ctx, t, "rgba32f", "fast")[0]
        exp = M.decode_full(t, NTHR)
        mx, mean = _err(got, exp)
        print(f"{name} t={t}: max {mx:.3e} mean {mean:.3e}")
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (name, t, mx, mean)


def test_fast_tiles_border_and_rgba8():
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed)
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    ids = [3, 1, 0, 2, 1]
    slots = [4, 0, 6, 2, 5]
    t = 0.3
    y32 = gpu_tiles(ctx, ids, t, "rgba32f", "fast", slots=slots, num_slots=8)
    q8 = gpu_tiles(ctx, ids, t, "rgba8", "fast", slots=slots, num_slots=8)
    exp = M.decode_tiles(ids, t, NTHR)
    for r, s in enumerate(slots):
        mx, mean = _err(y32[s], exp[r])
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (r, mx, mean)
        # RGBA8 = the oracle's fp32 quantiser applied to the kernel's own fp32 y
        np.testing.assert_array_equal(q8[s], oracle.quantize_rgba8(np.ascontiguousarray(y32[s])))
        dq = np.abs(q8[s][..., :3].astype(int) - oracle.quantize_rgba8(exp[r])[..., :3].astype(int))
        assert dq.max() <= 1
    # untouched slots stay zero
    assert (q8[1] == 0).all() and (q8[3] == 0).all() and (q8[7] == 0).all()


def test_fast_full_equals_tiles_core_and_deterministic():
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed, "mixed")
    ctx = _load(lay, th)
    full = gpu_full(ctx, 0.7, "rgba8")[0]
    full2 = gpu_full(ctx, 0.7, "rgba8")[0]
    np.testing.assert_array_equal(full, full2)
    tiles = gpu_tiles(ctx, [0, 1, 2, 3], 0.7, "rgba8")
    C, B = 128, 4
    for k in range(4):
        tx, ty = k % 2, k // 2
        np.testing.assert_array_equal(full[0, ty * C:(ty + 1) * C, tx * C:(tx + 1) * C], tiles[k, B:B + C, B:B + C])
        # mirrored border is an exact copy (R3)
        pad = np.pad(tiles[k, B:B + C, B:B + C], ((B, B), (B, B), (0, 0)), mode="reflect")
        np.testing.assert_array_equal(tiles[k], pad)


def test_cross_format_u8_equals_bc7():
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed, "mixed")
    lay8 = dict(lay, fmt_uv="u8", fmt_uvt="u8")
    th8 = dict(th)
    th8["uv"] = np.stack([oracle.bc7_decode_image(th["uv"][k].reshape(-1, 16), 128, 128) for k in range(4)])
    th8["uvt"] = np.stack([[oracle.bc7_decode_image(th["uvt"][k, d].reshape(-1, 16), 32, 32) for d in range(4)]
                           for k in range(4)])
    for mode in ("fast", "ref_fp32"):
        a = gpu_full(_load(lay, th), 0.45, "rgba32f", mode)
        b = gpu_full(_load(lay8, th8), 0.45, "rgba32f", mode)
        np.testing.assert_array_equal(a, b)


def _bcn_image(fmt, blocks, w, h):
    """Oracle decode of a [h/4][w/4] block map into [h][w][channels] u8."""
    nch = 2 if fmt == "bc5" else 4
    bsz = 8 if fmt == "bc1" else 16
    b = np.ascontiguousarray(blocks).reshape(h // 4, w // 4, bsz)
    out = np.zeros((h, w, nch), np.uint8)
    for by in range(h // 4):
        for bx in range(w // 4):
            out[4 * by:4 * by + 4, 4 * bx:4 * bx + 4] = oracle.bcn_decode_block(fmt, b[by, bx].tobytes()).reshape(4, 4, nch)
    return out


@pytest.mark.parametrize("fmt", ["bc1", "bc3"])
def test_cross_format_u8_equals_bcn(fmt):
    # the device BC1 / BC3 / BC5 decoders are bit-exact: decoding the same
    # blocks with the oracle into u8 maps gives identical outputs in both modes
    lay = S.layout(1, 2, 1, "M", uvt_depth=3, line_t=8, fmt_uv=fmt, fmt_uvt=fmt, fmt_line="bc5")
    th = S.make_theta(lay, 77, "mixed")
    lay8 = dict(lay, fmt_uv="u8", fmt_uvt="u8", fmt_line="u8")
    th8 = dict(th)
    R, R3, U, T = lay["uv_res"], lay["uvt_res"], lay["line_res"], lay["line_t"]
    th8["uv"] = np.stack([_bcn_image(fmt, th["uv"][k], R, R) for k in range(2)])
    th8["uvt"] = np.stack([[_bcn_image(fmt, th["uvt"][k, d], R3, R3) for d in range(3)] for k in range(2)])
    th8["ut"] = np.stack([_bcn_image("bc5", th["ut"][k], U, T) for k in range(2)])
    th8["vt"] = np.stack([_bcn_image("bc5", th["vt"][k], U, T) for k in range(2)])
    for mode in ("fast", "ref_fp32"):
        a = gpu_full(_load(lay, th), [0.45, 0.8], "rgba32f", mode)
        b = gpu_full(_load(lay8, th8), [0.45, 0.8], "rgba32f", mode)
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(gpu_tiles(_load(lay, th), [1, 0], 0.2, "rgba8"),
                                  gpu_tiles(_load(lay8, th8), [1, 0], 0.2, "rgba8"))


@pytest.mark.parametrize("fmt", ["bc1", "bc3"])
def test_ref_fp32_bcn(fmt):
    lay = S.layout(1, 2, 1, "M", uvt_depth=4, line_t=8, fmt_uv=fmt, fmt_uvt=fmt, fmt_line="bc5")
    th = S.make_theta(lay, 5, "smooth")
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    for t in (0.3, 0.9):
        mx, _ = _err(gpu_full(ctx, t, "rgba32f", "ref_fp32")[0], M.decode_full(t, NTHR))
        assert mx <= REF_MAX, (fmt, t, mx)


@pytest.mark.parametrize("payload", ["smooth", "mixed"])
def test_texture_unit_fetch_equals_software_decode(payload):
    # NDGI_MODE_FAST_TEXUNIT (F_uv through the texture unit's BC7 decoder) is
    # bit-identical to NDGI_MODE_FAST on all outputs, incl. all-mode payloads,
    # several atlases, decode_tiles with borders and small-batch strips
    lay = S.layout(2, 2, 2, "M", uvt_depth=4, line_t=4)
    th = S.make_theta(lay, 41, payload)
    ctx = _load(lay, th)
    for fmt in ("rgba8", "rgba32f"):
        np.testing.assert_array_equal(gpu_full(ctx, [0.2, 0.7], fmt, "fast_texunit"), gpu_full(ctx, [0.2, 0.7], fmt))
    ids = [5, 0, 7, 2]
    np.testing.assert_array_equal(gpu_tiles(ctx, ids, 0.33, "rgba8", "fast_texunit"), gpu_tiles(ctx, ids, 0.33, "rgba8"))
    np.testing.assert_array_equal(gpu_tiles(ctx, [3], 0.9, "rgba32f", "fast_texunit"), gpu_tiles(ctx, [3], 0.9))


def test_texture_unit_mode_needs_bc7():
    lay, seed = S.config("c1")
    lay8 = dict(lay, fmt_uv="u8")
    th = S.make_theta(lay8, seed)
    ctx = _load(lay8, th)
    with pytest.raises(ndgi.NdgiError) as e:
        gpu_full(ctx, 0.5, "rgba8", "fast_texunit")
    assert e.value.status == ndgi.ERR_UNSUPPORTED


def test_batch_equals_single_calls():
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed)
    ctx = _load(lay, th)
    ts = [i / 24 for i in range(0, 24, 3)]
    batch = gpu_full(ctx, ts, "rgba8")
    for i, t in enumerate(ts):
        np.testing.assert_array_equal(batch[i], gpu_full(ctx, t, "rgba8")[0])


def test_small_batches_strips():
    # n = 1 and n = 3 requests take the strip split (several units per tile)
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed)
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    for ids in ([2], [3, 0, 3]):
        got = gpu_tiles(ctx, ids, 0.9, "rgba32f")
        exp = M.decode_tiles(ids, 0.9, NTHR)
        mx, mean = _err(got, exp)
        assert mx <= FAST_MAX and mean <= FAST_MEAN


def test_windowed_uvt_small_strips():
    # H profile (windowed F_uvt) through decode_tiles: 4-row strips (n = 1),
    # 8-row strips and whole tiles, against the oracle
    lay = S.layout(1, 2, 2, "H")
    th = S.make_theta(lay, 17, "mixed")
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    for ids in ([1], [3, 0], list(range(4)) * 300):
        got = gpu_tiles(ctx, ids, 0.61, "rgba32f")
        exp = M.decode_tiles(ids[:4], 0.61, NTHR)
        mx, mean = _err(got[:4], exp)
        assert mx <= FAST_MAX and mean <= FAST_MEAN


def test_strip_split_is_bit_exact():
    # a tile decoded alone (4-row strips, 32 units) == the same tile inside a
    # batch big enough for whole-tile units (RGBA8 and RGBA32F, bit-equal)
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed)
    ctx = _load(lay, th)
    big = [k % 4 for k in range(2400)]
    for fmt in ("rgba8", "rgba32f"):
        many = gpu_tiles(ctx, big, 0.45, fmt)
        for k in range(4):
            one = gpu_tiles(ctx, [k], 0.45, fmt)
            np.testing.assert_array_equal(one[0], many[k])


def test_bad_ids_and_arguments():
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed)
    ctx = _load(lay, th)
    ndgi.ndgi_device_error(ctx, reset=True)
    out = gpu_tiles(ctx, [0, 7, 1], 0.5, "rgba8", slots=[0, 1, 9], num_slots=3)
    assert ndgi.ndgi_device_error(ctx, reset=True) == 2     # id 7 and slot 9 rejected
    assert (out[0] != 0).any() and (out[1] == 0).all()
    for mode in ("fast", "ref_fp32"):
        gpu_tiles(ctx, [5], 0.5, "rgba8", mode=mode)
        assert ndgi.ndgi_device_error(ctx, reset=True) == 1
    o = torch.zeros((4, 136, 136, 4), dtype=torch.uint8, device="cuda")
    ids = torch.zeros(4, dtype=torch.int32, device="cuda")
    for t in (float("nan"), -0.1, 1.5, float("inf")):
        with pytest.raises(ndgi.NdgiError) as e:
            ndgi.ndgi_decode_tiles(ctx, ids, None, 4, 4, t, o)
        assert e.value.status == ndgi.ERR_RANGE
    # an empty batch is an argument error (ndgi.h), not a launch
    with pytest.raises(ndgi.NdgiError) as e:
        ndgi.ndgi_decode_tiles(ctx, ids, None, 0, 4, 0.5, o)
    assert e.value.status == ndgi.ERR_ARG
    lay_bad = dict(lay, hidden=8)
    th_bad = S.make_theta(lay_bad, 1)
    ctx_bad = _load(lay_bad, th_bad)
    with pytest.raises(ndgi.NdgiError) as e:
        ndgi.ndgi_decode_full(ctx_bad, 0.5, o, "rgba8", "fast")
    assert e.value.status == ndgi.ERR_UNSUPPORTED


def test_c2_fullsize_sampled():
    """Config 2 (4096^2 atlas, 1024 tiles) in the bench's launch configuration:
    sampled texels against the oracle evaluated one by one, two whole tiles."""
    lay, seed = S.config("c2")
    th = S.make_theta(lay, seed)
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    ts = [5 / 24, 17 / 24]
    got = gpu_full(ctx, ts, "rgba32f")
    rng = np.random.default_rng(0)
    C = 128
    for ti, t in enumerate(ts):
        errs = []
        for _ in range(400):
            k = int(rng.integers(0, 1024))
            i, j = (int(v) for v in rng.integers(0, C, 2))
            tx, ty = k % 32, k // 32
            exp = M.texel(k, i + 4, j + 4, t)
            errs.append(np.abs(got[ti, 0, ty * C + j, tx * C + i, :3] - exp))
        errs = np.array(errs)
        assert errs.max() <= FAST_MAX and errs.mean() <= FAST_MEAN
        for k in (0, 1023):
            tx, ty = k % 32, k // 32
            exp = M.decode_tiles([k], t, NTHR)[0, 4:4 + C, 4:4 + C]
            mx, mean = _err(got[ti, 0, ty * C:(ty + 1) * C, tx * C:(tx + 1) * C], exp)
            assert mx <= FAST_MAX and mean <= FAST_MEAN


@pytest.mark.parametrize("name", ["c5:M:bc3", "c5:M:bc1", "c5:H:bc3", "c5:M64:bc7"])
def test_c5_fullsize_sampled(name):
    """Config 5 cells at full size (c2's 1,024-tile atlas), four times per call
    (RGBA8 and RGBA32F): sampled texels against the oracle one by one; RGBA8 =
    the oracle's quantiser of the kernel's own fp32 output."""
    lay, seed = S.config(name)
    th = S.make_theta(lay, seed)
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    ts = [i / 24 for i in (0, 7, 13, 23)]
    y32 = gpu_full(ctx, ts, "rgba32f")
    q8 = gpu_full(ctx, ts, "rgba8")
    rng = np.random.default_rng(3)
    C = 128
    errs = []
    for _ in range(150):
        ti = int(rng.integers(0, len(ts)))
        k = int(rng.integers(0, 1024))
        i, j = (int(v) for v in rng.integers(0, C, 2))
        tx, ty = k % 32, k // 32
        exp = M.texel(k, i + 4, j + 4, ts[ti])
        got = y32[ti, 0, ty * C + j, tx * C + i]
        errs.append(np.abs(got[:3] - exp))
        np.testing.assert_array_equal(q8[ti, 0, ty * C + j, tx * C + i],
                                      oracle.quantize_rgba8(np.ascontiguousarray(got[None]))[0])
    errs = np.array(errs)
    assert errs.max() <= FAST_MAX and errs.mean() <= FAST_MEAN, (name, errs.max(), errs.mean())


def test_c2_bench_launch_all_texels_of_one_time():
    """The exact launch bench.py times (config 2, decode_full_batch over the 24
    times, RGBA8, the FULL8 kernel): every texel of one time against the
    oracle's own RGBA8 quantisation (<= 1 level, R12), and 100 sampled texels of
    each of the other 23 times."""
    lay, seed = S.config("c2")
    th = S.make_theta(lay, seed)
    M = oracle.Model(lay, th)
    ctx = _load(lay, th)
    ts = [i / 24 for i in range(24)]
    q = gpu_full(ctx, ts, "rgba8")                        # [24][1][4096][4096][4]
    t_full = 13
    exp = oracle.quantize_rgba8(M.decode_full(ts[t_full], NTHR).reshape(-1, 3)).reshape(q.shape[1:])
    d = np.abs(q[t_full].astype(int) - exp.astype(int))
    assert d.max() <= 1 and (d[..., 3] == 0).all()
    assert (d[..., :3] == 0).mean() > 0.99
    rng = np.random.default_rng(7)
    C = 128
    for ti, t in enumerate(ts):
        if ti == t_full:
            continue
        for _ in range(100):
            k = int(rng.integers(0, 1024))
            i, j = (int(v) for v in rng.integers(0, C, 2))
            tx, ty = k % 32, k // 32
            e = oracle.quantize_rgba8(M.texel(k, i + 4, j + 4, t).reshape(1, 3))[0]
            g = q[ti, 0, ty * C + j, tx * C + i]
            assert np.abs(g.astype(int) - e.astype(int)).max() <= 1


@pytest.mark.parametrize("cell", ["c2", "c5:H:bc7"])
def test_dynamic_schedule_and_tail_strips_equal_single_calls(cell):
    """A 24-t decode_full_batch of 1,024 tiles has more units than resident CTAs:
    units are claimed dynamically and the last ~1,184 (t, tile) jobs run as
    4 strips each (KParams::tail_from).  Every byte must equal the single-t
    calls, which run one whole-tile unit per CTA (static)."""
    lay, seed = S.config(cell)
    ctx = _load(lay, S.make_theta(lay, seed))
    ts = [i / 24 for i in range(24)]
    q = gpu_full(ctx, ts, "rgba8")
    for ti in (0, 7, 21, 22, 23):
        np.testing.assert_array_equal(q[ti], gpu_full(ctx, ts[ti], "rgba8")[0])


def test_dynamic_schedule_with_invalid_requests():
    """A decode_tiles batch with more units than resident CTAs (1,200 requests
    -> 4 strips each, claimed dynamically) in which every 7th id and every 11th
    slot is invalid: the skipped units still claim their successors (no unit
    lost, no hang), the error counter counts each bad request once, and every
    valid slot is byte-identical to the same tile decoded alone."""
    lay, seed = S.config("c1")
    ctx = _load(lay, S.make_theta(lay, seed))
    n = 1200
    rng = np.random.default_rng(5)
    ids = rng.integers(0, 4, n)
    ids[::7] = 4 + (np.arange(len(ids[::7])) % 3)          # id >= num_tiles
    slots = np.arange(n)
    slots[5::11] = n + 3                                     # slot >= num_slots
    bad = (ids >= 4) | (slots >= n)
    ndgi.ndgi_device_error(ctx, reset=True)
    out = gpu_tiles(ctx, ids, 0.45, "rgba8", slots=slots, num_slots=n)
    assert ndgi.ndgi_device_error(ctx, reset=True) == int(bad.sum())
    alone = {k: gpu_tiles(ctx, [k], 0.45, "rgba8")[0] for k in range(4)}
    for r in range(n):
        if bad[r]:
            if slots[r] < n:
                assert (out[slots[r]] == 0).all(), r
        else:
            np.testing.assert_array_equal(out[slots[r]], alone[int(ids[r])], err_msg=str(r))


def test_host_buffer_path():
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed)
    ctx = _load(lay, th)
    ts = [0.1, 0.2, 0.3]
    host = torch.zeros((3, 1, 256, 256, 4), dtype=torch.uint8).pin_memory()
    ndgi.ndgi_decode_full_host(ctx, ts, host, "rgba8")
    np.testing.assert_array_equal(host.numpy(), gpu_full(ctx, ts, "rgba8"))


def _tile_oracle(seed, k, t):
    """Oracle decode of global tile k alone (payloads depend only on (seed, k))."""
    lay1 = S.layout(1, 1, 1, "M")
    return oracle.Model(lay1, S.make_theta(lay1, seed, tiles=[k])).decode_tiles([0], t, NTHR)[0, 4:132, 4:132]


def test_c4_full_scene_one_gpu_sampled():
    """Config 4's whole 16,384-tile scene (4 x 8192^2 atlases, the maximum size)
    in one decode_full call, RGBA8 and RGBA32F: sampled texels of the GPU output
    against the oracle evaluated per global tile id."""
    lay, seed = S.config("c4")
    th = S.make_theta(lay, seed)
    ctx = _load(lay, th)
    t = 11 / 24
    y = gpu_full(ctx, t, "rgba32f")[0]              # [4][8192][8192][4]
    q = gpu_full(ctx, t, "rgba8")[0]
    C = 128
    rng = np.random.default_rng(11)
    for k in [0, 16383, *rng.integers(1, 16383, 4).tolist()]:
        a, r = divmod(int(k), 64 * 64)
        ty, tx = divmod(r, 64)
        exp = _tile_oracle(seed, int(k), t)
        got = y[a, ty * C:(ty + 1) * C, tx * C:(tx + 1) * C]
        mx, mean = _err(got, exp)
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (k, mx, mean)
        np.testing.assert_array_equal(q[a, ty * C:(ty + 1) * C, tx * C:(tx + 1) * C],
                                      oracle.quantize_rgba8(np.ascontiguousarray(got)))


@pytest.mark.parametrize("rank", [0, 5])
def test_c4_shard_of_eight_matches_global_tiles(rank):
    """bench.py --workload c4 at N = 8: rank r holds tiles k % 8 == r in a
    compact 64 x 32 atlas; each local tile l must equal the oracle's decode of
    global tile shard_tiles(...)[l] (no hot-path communication needed)."""
    from paper_2604_12625_b200 import parallel as par
    _, seed = S.config("c4")
    gids = par.shard_tiles(16384, 8, rank)
    lay = S.layout(1, 64, len(gids) // 64, "M")
    ctx = _load(lay, S.make_theta(lay, seed, tiles=gids))
    t = 19 / 24
    y = gpu_full(ctx, t, "rgba32f")[0, 0]
    C = 128
    rng = np.random.default_rng(rank)
    for l in [0, len(gids) - 1, *rng.integers(1, len(gids) - 1, 3).tolist()]:
        ty, tx = divmod(int(l), 64)
        mx, mean = _err(y[ty * C:(ty + 1) * C, tx * C:(tx + 1) * C], _tile_oracle(seed, int(gids[l]), t))
        assert mx <= FAST_MAX and mean <= FAST_MEAN, (rank, l, mx, mean)
