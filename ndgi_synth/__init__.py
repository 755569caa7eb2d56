"""Seeded synthetic inputs for the NDGI tile decode: layouts and Theta payloads.

This module is shared by the tests, the bench and the oracle wrappers, and
holds NONE of the method's arithmetic: it never decodes BC7, samples a map,
evaluates gamma(t) or runs the MLP.  It only *writes* bit patterns (BC7
blocks are packed from chosen endpoint/index fields), u8/f16 maps and f16
weights, from a counter-based hash so that any subset of tiles can be
generated independently (tile k's payload depends only on (seed, k)).

Recipe:
* geometry and profiles from the paper: Table 1, Table 3
  (P:245-250), VT tiles of 128^2 with a 4-texel border;
* BC7 "smooth" payload (default): mode-6 blocks whose endpoints bracket a
  smooth per-channel field 0.5 + 0.3 sin(2 pi (a x + b y) + phi) at block
  resolution (+-delta, delta in [0.02, 0.12]); per-texel 4-bit indices are
  hashed noise.  This matches what BC simulation trains toward (one
  endpoint pair + per-texel weights, Eq. 6-7);
* BC7 "mixed" payload: mode m uniform in 0..7 forced through byte 0, all
  other bits random (bit-exactness stress, worst-case divergence);
* U8 / F16 maps: the smooth field quantised to u8 (F16 = fp16(q/255));
* line maps F_ut / F_vt: smooth u8 fields over (space, time), [T][U][2];
* BC1 / BC3 / BC5 payloads (R29, config 5's BC-format axis): endpoints
  bracket the same smooth field at block resolution (+-delta), endpoint
  order hashed (both BC1 colour modes, both BC4 palettes), indices hashed;
  "mixed" = all bits random;
* MLP: PyTorch nn.Linear default init U(+-1/sqrt(fan_in)) for W and b,
  b3 += 0.5, rounded to f16 (R11); mlp="stress" scales the layers (see
  MLP_SCALES) so the hidden pre-activations reach |z| ~ 10 and the outputs
  leave [0, 1] on both sides.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

PROFILES = {  # Table 3: F_uvt resolution and hidden size
    "L": dict(uvt_res=16, hidden=16),
    "M": dict(uvt_res=32, hidden=16),
    "H": dict(uvt_res=64, hidden=16),
    "M64": dict(uvt_res=32, hidden=64),
}


def layout(atlases=1, tiles_x=1, tiles_y=1, profile="M", core=128, border=4, uv_res=None,
           uvt_depth=12, line_res=64, line_t=24, fmt_uv="bc7", fmt_uvt="bc7", fmt_line="u8",
           gelu="erf", border_mode="mirror", hidden=None, uvt_res=None) -> dict:
    p = PROFILES[profile]
    return dict(
        num_tiles=atlases * tiles_x * tiles_y, atlases=atlases, tiles_x=tiles_x, tiles_y=tiles_y,
        core=core, border=border, uv_res=core if uv_res is None else uv_res,
        uvt_res=p["uvt_res"] if uvt_res is None else uvt_res, uvt_depth=uvt_depth,
        line_res=line_res, line_t=line_t, hidden=p["hidden"] if hidden is None else hidden,
        fmt_uv=fmt_uv, fmt_uvt=fmt_uvt, fmt_line=fmt_line, gelu=gelu, border_mode=border_mode)


def config(name: str) -> tuple[dict, int]:
    """The five BASELINE.json configs as (layout, seed).

    c1: one 256^2 lightmap = 2x2 tiles, few keyframes (D=4, T=4), profile M
    c2: one 4096^2 atlas = 32x32 tiles, profile M (Table 1 shapes)
    c3/c4: 4 x 8192^2 atlases = 16384 tiles, profile M (FarmLand scale)
    c5:<profile>:<fmt>: c2's atlas with profile in {L,M,H,M64}, fmt in {bc7,bc3,bc1,u8,f16}
        (line maps: u8 with bc7, BC5 with bc3 / bc1, else the same format)
    """
    if name == "c1":
        return layout(1, 2, 2, "M", uvt_depth=4, line_t=4), 1000
    if name == "c2":
        return layout(1, 32, 32, "M"), 2000
    if name == "c3":
        return layout(4, 64, 64, "M"), 3000
    if name == "c4":
        return layout(4, 64, 64, "M"), 4000
    if name.startswith("c5"):
        _, prof, fmt = name.split(":")
        line = {"bc7": "u8", "bc1": "bc5", "bc3": "bc5"}.get(fmt, fmt)
        return layout(1, 32, 32, prof, fmt_uv=fmt, fmt_uvt=fmt, fmt_line=line), 5000
    raise KeyError(name)


# ------------------------------------------------------------------ hashing
def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _tile_keys(seed: int, stream: int, tiles: np.ndarray) -> np.ndarray:
    base = np.uint64((seed * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF) ^ np.uint64(stream << 40)
    return splitmix64(base ^ tiles.astype(np.uint64))


def _hash(keys: np.ndarray, n: int) -> np.ndarray:
    """[tiles] keys -> [tiles][n] uint64 random words."""
    idx = np.arange(n, dtype=np.uint64)
    return splitmix64(keys[:, None] ^ splitmix64(idx)[None, :])


def _unif(words: np.ndarray) -> np.ndarray:
    return (words >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


# ------------------------------------------------------------------ fields
def _field_params(seed, stream, tiles, nch):
    w = _unif(_hash(_tile_keys(seed, stream, tiles), 3 * nch)).reshape(len(tiles), nch, 3)
    a = 0.5 + 2.5 * w[..., 0]
    b = 0.5 + 2.5 * w[..., 1]
    phi = 2 * np.pi * w[..., 2]
    return a, b, phi


def _smooth(a, b, phi, xs, ys):
    """[tiles][ch] params, xs/ys normalised coords [...] -> [tiles][...][ch] (float32)."""
    arg = 2 * np.pi * (a[:, None, :] * xs.reshape(1, -1, 1) + b[:, None, :] * ys.reshape(1, -1, 1)) + phi[:, None, :]
    return 0.5 + 0.3 * np.sin(arg.astype(np.float32))


def _smooth_grid(a, b, phi, n):
    """Separable evaluation of _smooth on the n x n grid of cell centres:
    sin(X + Y) = sin X cos Y + cos X sin Y.  -> [tiles][n*n][ch] float32."""
    c = ((np.arange(n) + 0.5) / n).astype(np.float32)
    X = 2 * np.pi * a[:, None, :].astype(np.float32) * c[None, :, None]                  # [t][n][ch]
    Y = 2 * np.pi * b[:, None, :].astype(np.float32) * c[None, :, None] + phi[:, None, :].astype(np.float32)
    sx, cx, sy, cy = np.sin(X), np.cos(X), np.sin(Y), np.cos(Y)
    v = sy[:, :, None, :] * cx[:, None, :, :] + cy[:, :, None, :] * sx[:, None, :, :]  # [t][y][x][ch]
    return (0.5 + 0.3 * v).reshape(a.shape[0], n * n, a.shape[1])


class _BitPacker:
    """Packs LSB-first fields into 128-bit blocks (two uint64 words)."""

    def __init__(self, shape):
        self.lo = np.zeros(shape, np.uint64)
        self.hi = np.zeros(shape, np.uint64)
        self.pos = 0

    def put(self, v, width):
        v = np.asarray(v).astype(np.uint64) & np.uint64((1 << width) - 1)
        p = self.pos
        if p + width <= 64:
            self.lo |= v << np.uint64(p)
        elif p >= 64:
            self.hi |= v << np.uint64(p - 64)
        else:
            self.lo |= v << np.uint64(p)
            self.hi |= v >> np.uint64(64 - p)
        self.pos += width

    def bytes(self):
        assert self.pos == 128, self.pos
        out = np.empty(self.lo.shape + (16,), np.uint8)
        out[..., :8] = self.lo[..., None].view(np.uint8).reshape(self.lo.shape + (8,))
        out[..., 8:] = self.hi[..., None].view(np.uint8).reshape(self.hi.shape + (8,))
        return out


def bc7_mode6_blocks(lo8: np.ndarray, hi8: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Pack mode-6 blocks.  lo8/hi8: [...,4] 8-bit endpoint targets; idx: [...,16] 4-bit.

    Field order (D3D11 BC7 mode 6): mode bits 0000001, R0 R1 G0 G1 B0 B1 A0 A1
    (7 bits each), P0, P1, then 16 indices (texel 0 has 3 bits, anchor)."""
    shape = lo8.shape[:-1]
    bp = _BitPacker(shape)
    bp.put(np.full(shape, 1 << 6), 7)
    for c in range(4):
        bp.put(lo8[..., c] >> 1, 7)
        bp.put(hi8[..., c] >> 1, 7)
    bp.put(np.zeros(shape), 1)   # P0 = 0
    bp.put(np.ones(shape), 1)    # P1 = 1
    bp.put(idx[..., 0] & 7, 3)
    for i in range(1, 16):
        bp.put(idx[..., i], 4)
    return bp.bytes()


def bc7_random_blocks(words: np.ndarray, modes: np.ndarray) -> np.ndarray:
    """[..., 2] random uint64 words + [...] modes (0..8) -> [...,16] blocks."""
    out = np.empty(words.shape[:-1] + (16,), np.uint8)
    out[..., :8] = words[..., 0:1].view(np.uint8).reshape(words.shape[:-1] + (8,))
    out[..., 8:] = words[..., 1:2].view(np.uint8).reshape(words.shape[:-1] + (8,))
    m = modes.astype(np.int64)
    b0 = out[..., 0].astype(np.int64)
    keep = np.where(m >= 7, 0, (0xFF << (m + 1)) & 0xFF)
    b0 = np.where(m >= 8, 0, (b0 & keep) | (1 << np.minimum(m, 7)))
    out[..., 0] = b0.astype(np.uint8)
    return out


def _bc7_map(seed, stream, tiles, R, nslices, payload):
    """[tiles][nslices][R/4][R/4][16] BC7 blocks."""
    nb = R // 4
    nblk = nslices * nb * nb
    if payload == "mixed":
        keys = _tile_keys(seed, stream, tiles)
        words = _hash(keys, 3 * nblk).reshape(len(tiles), nblk, 3)
        modes = (words[..., 2] % np.uint64(8)).astype(np.int64)
        blk = bc7_random_blocks(words[..., :2], modes)
        return blk.reshape(len(tiles), nslices, nb, nb, 16)
    a, b, phi = _field_params(seed, stream, tiles, 4)
    out = np.empty((len(tiles), nslices, nb, nb, 16), np.uint8)
    keys = _tile_keys(seed, stream + 100, tiles)
    words = _hash(keys, 2 * nblk).reshape(len(tiles), nslices, nb * nb, 2)
    for s in range(nslices):
        m = _smooth_grid(a, b, phi + 0.7 * s, nb)            # [tiles][nb*nb][4]
        d = (0.02 + 0.10 * _unif(words[:, s, :, 0])[..., None]).astype(np.float32)
        lo = np.clip(np.rint((m - d) * 255), 0, 255).astype(np.uint64)
        hi = np.clip(np.rint((m + d) * 255), 0, 255).astype(np.uint64)
        # mode 6: bits 0..6 mode, then R0 R1 G0 G1 B0 B1 A0 A1 (7 bits each), P0 = 0 (bit 63);
        # second word: P1 = 1 (bit 0), indices (bits 1..63) = hashed noise
        w0 = np.full(lo.shape[:-1], 1 << 6, np.uint64)
        for c in range(4):
            w0 |= (lo[..., c] >> np.uint64(1)) << np.uint64(7 + 14 * c)
            w0 |= (hi[..., c] >> np.uint64(1)) << np.uint64(14 + 14 * c)
        w1 = words[:, s, :, 1] | np.uint64(1)
        blk = np.stack([w0, w1], -1).view(np.uint8)
        out[:, s] = blk.reshape(len(tiles), nb, nb, 16)
    return out


BCN_BLOCK_BYTES = {"bc1": 8, "bc3": 16, "bc5": 16}


def _bcn_map(seed, stream, tiles, rx, ry, nslices, fmt, payload):
    """[tiles][nslices][ry/4][rx/4][8 or 16] BC1 / BC3 / BC5 blocks (layouts
    in include/ndgi.h): packed from chosen endpoints and hashed indices."""
    nbx, nby = rx // 4, ry // 4
    nb = nbx * nby
    bsz = BCN_BLOCK_BYTES[fmt]
    nw = bsz // 8
    keys = _tile_keys(seed, stream + 200, tiles)
    if payload == "mixed":
        w = _hash(keys, nslices * nb * nw)
        return w.view(np.uint8).reshape(len(tiles), nslices, nby, nbx, bsz)
    nch = 2 if fmt == "bc5" else 4
    a, b, phi = _field_params(seed, stream, tiles, nch)
    xs = np.tile((np.arange(nbx) + 0.5) / nbx, nby)
    ys = np.repeat((np.arange(nby) + 0.5) / nby, nbx)
    out = np.empty((len(tiles), nslices, nb, nw), np.uint64)
    words = _hash(keys, nslices * nb * 4).reshape(len(tiles), nslices, nb, 4)
    for s in range(nslices):
        m = _smooth(a, b, phi + 0.7 * s, xs, ys)                       # [tiles][nb][nch]
        d = (0.02 + 0.10 * _unif(words[:, s, :, 0])[..., None]).astype(np.float32)
        lo = np.clip(np.rint((m - d) * 255), 0, 255).astype(np.uint64)
        hi = np.clip(np.rint((m + d) * 255), 0, 255).astype(np.uint64)
        sw = words[:, s, :, 1]                                         # endpoint-order bits

        def bc4(c, bit):
            e0, e1 = lo[..., c], hi[..., c]
            swap = ((sw >> np.uint64(bit)) & np.uint64(1)).astype(bool)
            a0, a1 = np.where(swap, e1, e0), np.where(swap, e0, e1)
            return a0 | (a1 << np.uint64(8)) | ((words[:, s, :, 2 + (bit & 1)] >> np.uint64(16)) << np.uint64(16))

        def bc1():
            c = [(lo[..., 0] >> np.uint64(3) << np.uint64(11)) | (lo[..., 1] >> np.uint64(2) << np.uint64(5)) |
                 (lo[..., 2] >> np.uint64(3)),
                 (hi[..., 0] >> np.uint64(3) << np.uint64(11)) | (hi[..., 1] >> np.uint64(2) << np.uint64(5)) |
                 (hi[..., 2] >> np.uint64(3))]
            swap = (sw & np.uint64(1)).astype(bool)
            c0, c1 = np.where(swap, c[1], c[0]), np.where(swap, c[0], c[1])
            return c0 | (c1 << np.uint64(16)) | ((words[:, s, :, 2] >> np.uint64(32)) << np.uint64(32))

        if fmt == "bc1":
            out[:, s, :, 0] = bc1()
        elif fmt == "bc3":
            out[:, s, :, 0] = bc4(3, 1)
            out[:, s, :, 1] = bc1()
        else:
            out[:, s, :, 0] = bc4(0, 2)
            out[:, s, :, 1] = bc4(1, 3)
    return out.view(np.uint8).reshape(len(tiles), nslices, nby, nbx, bsz)


def _dense_map(seed, stream, tiles, rx, ry, nch, nslices, fmt):
    """[tiles][nslices][ry][rx][nch] u8 (or f16 of q/255) smooth field."""
    a, b, phi = _field_params(seed, stream, tiles, nch)
    xs = np.tile((np.arange(rx) + 0.5) / rx, ry)
    ys = np.repeat((np.arange(ry) + 0.5) / ry, rx)
    keys = _tile_keys(seed, stream + 100, tiles)
    out = np.empty((len(tiles), nslices, ry, rx, nch), np.uint8)
    for s in range(nslices):
        f = _smooth(a, b, phi + 0.7 * s, xs, ys)
        noise = _unif(_hash(keys ^ np.uint64(s), rx * ry * nch)).reshape(len(tiles), rx * ry, nch) - 0.5
        out[:, s] = np.clip(np.rint((f + 0.1 * noise) * 255), 0, 255).astype(np.uint8).reshape(len(tiles), ry, rx, nch)
    if fmt == "f16":
        return (out.astype(np.float64) / 255.0).astype(np.float16)
    return out


# "stress" MLP (GPU parity outside the seeded regime): W1, b1 x 6, W2, b2 x 2.5,
# W3, b3 x 0.4 and b3 shifted by 0.5 + 0.4 U(-1, 1) per tile and channel, so
# that hidden pre-activations reach |z| ~ 9-11 and ~10 % of the outputs fall
# below 0 and ~12 % above 1 (the RGBA8 clamp of R12 on both sides)
MLP_SCALES = {"default": (1.0, 1.0, 1.0, 0.0), "stress": (6.0, 2.5, 0.4, 0.4)}


def _mlp(seed, tiles, h, kind="default"):
    keys = _tile_keys(seed, 5, tiles)
    n = 16 * h + h + h * h + h + 3 * h + 3
    u = _unif(_hash(keys, n + 3)) * 2.0 - 1.0               # U(-1, 1)
    s1, s2, s3, sb = MLP_SCALES[kind]
    sizes = [(16 * h, 16, s1), (h, 16, s1), (h * h, h, s2), (h, h, s2), (3 * h, h, s3), (3, h, s3)]  # (count, fan_in, scale)
    parts, o = [], 0
    for cnt, fan, sc in sizes:
        parts.append(u[:, o:o + cnt] / np.sqrt(fan) * sc)
        o += cnt
    w = np.concatenate(parts, axis=1)
    w[:, -3:] += 0.5 + sb * u[:, n:n + 3]
    return w.astype(np.float16).view(np.uint16)


def make_theta(lay: dict, seed: int, payload: str = "smooth", tiles=None, mlp: str = "default") -> dict:
    """Theta arrays for tile ids `tiles` (default all) in the layout's formats.

    Returns numpy arrays: uv, uvt, ut, vt (uint8 or float16) and mlp (uint16
    f16 bit patterns), each with the tile axis first, in the dense per-tile
    layouts that include/ndgi.h documents."""
    tiles = np.arange(lay["num_tiles"], dtype=np.int64) if tiles is None else np.asarray(tiles, np.int64)
    R, R3, D = lay["uv_res"], lay["uvt_res"], lay["uvt_depth"]
    th = {}
    if lay["fmt_uv"] == "bc7":
        th["uv"] = _bc7_map(seed, 1, tiles, R, 1, payload).reshape(len(tiles), R // 4, R // 4, 16)
    elif lay["fmt_uv"] in BCN_BLOCK_BYTES:
        th["uv"] = _bcn_map(seed, 1, tiles, R, R, 1, lay["fmt_uv"], payload)[:, 0]
    else:
        th["uv"] = _dense_map(seed, 1, tiles, R, R, 4, 1, lay["fmt_uv"]).reshape(len(tiles), R, R, 4)
    if lay["fmt_uvt"] == "bc7":
        th["uvt"] = _bc7_map(seed, 2, tiles, R3, D, payload)
    elif lay["fmt_uvt"] in BCN_BLOCK_BYTES:
        th["uvt"] = _bcn_map(seed, 2, tiles, R3, R3, D, lay["fmt_uvt"], payload)
    else:
        th["uvt"] = _dense_map(seed, 2, tiles, R3, R3, 4, D, lay["fmt_uvt"])
    U, T = lay["line_res"], lay["line_t"]
    if lay["fmt_line"] == "bc5":
        th["ut"] = _bcn_map(seed, 3, tiles, U, T, 1, "bc5", payload)[:, 0]
        th["vt"] = _bcn_map(seed, 4, tiles, U, T, 1, "bc5", payload)[:, 0]
    else:
        th["ut"] = _dense_map(seed, 3, tiles, U, T, 2, 1, lay["fmt_line"]).reshape(len(tiles), T, U, 2)
        th["vt"] = _dense_map(seed, 4, tiles, U, T, 2, 1, lay["fmt_line"]).reshape(len(tiles), T, U, 2)
    th["mlp"] = _mlp(seed, tiles, lay["hidden"], mlp)
    return th


def theta_bytes(lay: dict) -> int:
    """Whole-Theta bytes per tile (all t), for BPP accounting."""
    def b2(fmt, rx, ry, nc):
        if fmt == "bc7" or fmt in BCN_BLOCK_BYTES:
            return (rx // 4) * (ry // 4) * BCN_BLOCK_BYTES.get(fmt, 16)
        return rx * ry * nc * (1 if fmt == "u8" else 2)
    h = lay["hidden"]
    return (b2(lay["fmt_uv"], lay["uv_res"], lay["uv_res"], 4)
            + lay["uvt_depth"] * b2(lay["fmt_uvt"], lay["uvt_res"], lay["uvt_res"], 4)
            + 2 * b2(lay["fmt_line"], lay["line_res"], lay["line_t"], 2)
            + 2 * (16 * h + h + h * h + h + 3 * h + 3))


def vt_batches(num_tiles: int, n: int, frames: int, seed: int = 3000):
    """Config 3: per frame f, n distinct tile ids uniform without replacement,
    t_f = frac(0.3 + f/96) (one time bucket per frame)."""
    out = []
    for f in range(frames):
        keys = splitmix64(np.uint64(seed + f) ^ splitmix64(np.arange(num_tiles, dtype=np.uint64)))
        ids = np.argsort(keys, kind="stable")[:n].astype(np.uint32)
        out.append((ids, (0.3 + f / 96.0) % 1.0))
    return out


# ------------------------------------------------------------------ shading side (NEXT 1)
def page_cache_bytes(slots: int, core: int, border: int, seed: int) -> np.ndarray:
    """Seeded random RGBA8 page cache [slots][P][P][4] (A = 255)."""
    P = core + 2 * border
    words = splitmix64(np.arange(slots * P * P, dtype=np.uint64) + np.uint64(seed) * np.uint64(0x9E3779B9))
    rgba = words.view(np.uint8).reshape(slots * P * P, 8)[:, :4].copy()
    rgba[:, 3] = 255
    return rgba.reshape(slots, P, P, 4)


def hdr_params(atlases: int, n_frames: int, seed: int, gamma: float = 2.2):
    """Bake times i/(n_frames-1) (hourly bakes over t in [0,1]) and seeded
    per-atlas, per-time, per-channel means in [0.2, 8]."""
    times = np.linspace(0.0, 1.0, n_frames).astype(np.float32)
    w = splitmix64(np.arange(atlases * n_frames * 3, dtype=np.uint64) + np.uint64(seed))
    means = (0.2 + 7.8 * _unif(w)).astype(np.float32).reshape(atlases, n_frames, 3)
    return gamma, times, means


def shading_uv(n: int, seed: int, coherent: bool = False, width: int = 1920, height: int = 1080) -> np.ndarray:
    """Sample positions [n][2] float32: uniform random over [0,1]^2, or a
    screen-like coherent raster (a width x height grid over a sub-rectangle)."""
    if not coherent:
        w = splitmix64(np.arange(2 * n, dtype=np.uint64) + np.uint64(seed))
        return _unif(w).astype(np.float32).reshape(n, 2)
    ys, xs = np.mgrid[0:height, 0:width]
    u = 0.1 + 0.5 * (xs.ravel() + 0.5) / width
    v = 0.2 + 0.5 * (ys.ravel() + 0.5) / height
    uv = np.stack([u, v], 1).astype(np.float32)
    return np.resize(uv, (n, 2))


# ------------------------------------------------------------------ fine-tuning (NEXT 4)
def train_batch(tiles, S: int, seed: int, n_times: int = 24):
    """Seeded training samples for each tile: (u, v) at random texel centres of
    a 128^2 core, t at one of n_times bake times (P:531 hourly bakes), and a
    synthetic target lightmap value per sample: a smooth per-tile RGB field that
    drifts with t (values in [0.1, 0.9]).  Returns float32 samples, targets [n][S][3]."""
    tiles = np.asarray(tiles, np.int64)
    n = len(tiles)
    keys = _tile_keys(seed, 77, tiles)
    w = splitmix64(keys[:, None] * np.uint64(0x100000001B3) + np.arange(3 * S, dtype=np.uint64)[None, :])
    r = _unif(w).reshape(n, S, 3)
    i = np.floor(r[..., 0] * 128)
    j = np.floor(r[..., 1] * 128)
    f = np.floor(r[..., 2] * n_times)
    u, v, t = (i + 0.5) / 128, (j + 0.5) / 128, f / n_times
    pw = _unif(splitmix64(keys[:, None] + np.arange(9, dtype=np.uint64)[None, :] * np.uint64(0x9E37)))   # [n][9]
    tg = np.stack([0.5 + 0.4 * np.sin(2 * np.pi * ((0.5 + 2 * pw[:, None, c]) * u + (0.5 + 2 * pw[:, None, 3 + c]) * v
                                                    + pw[:, None, 6 + c] + 0.5 * t)) for c in range(3)], -1)
    return np.stack([u, v, t], -1).astype(np.float32), tg.astype(np.float32)
