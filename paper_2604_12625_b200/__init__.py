"""Python binding of libndgi.so -- the B200-native NDGI tile decoder.

Argument marshalling only: every step of the decode runs in the CUDA kernels
behind the C ABI declared in ``include/ndgi.h`` (functions of the same names
below).  PyTorch is used only to hold device memory and streams.  There is no
CPU fallback: importing this package without the built library raises.

    import paper_2604_12625_b200 as ndgi
    ctx = ndgi.ndgi_load(layout_dict, theta_tensors_on_cuda, device=0)
    ndgi.ndgi_decode_tiles(ctx, ids, None, n, num_slots, t, out_cache)
    ndgi.ndgi_decode_full(ctx, t, out)
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NDGI_LIB") or os.path.join(_HERE, "libndgi.so")   # NDGI_LIB: experiment builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2604_12625_b200/build.py` "
        "(or __graft_entry__.build()); there is no fallback implementation")

_lib = C.CDLL(LIB_PATH)

ABI_VERSION = 1
OK, ERR_ARG, ERR_RANGE, ERR_UNSUPPORTED, ERR_CUDA, ERR_NOMEM, ERR_DEVICE = range(7)
FMT = {"bc7": 0, "u8": 1, "f16": 2, "bc1": 3, "bc3": 4, "bc5": 5}
OUT = {"rgba8": 0, "rgba16f": 1, "rgba32f": 2}
GELU = {"erf": 0, "tanh": 1}
BORDER = {"mirror": 0, "eval_clamp": 1}
MODE = {"fast": 0, "ref_fp32": 1, "fast_texunit": 2}
TEXEL_BYTES = {"rgba8": 4, "rgba16f": 8, "rgba32f": 16}


class ndgi_layout(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "abi_version", "num_tiles", "atlases", "tiles_x", "tiles_y", "core", "border", "uv_res",
        "uvt_res", "uvt_depth", "line_res", "line_t", "hidden", "fmt_uv", "fmt_uvt", "fmt_line",
        "gelu", "border_mode")]


class ndgi_hdr(C.Structure):
    _fields_ = [("gamma", C.c_float), ("n_frames", C.c_uint32), ("frame_times", C.c_void_p), ("means", C.c_void_p)]


class ndgi_params(C.Structure):
    _fields_ = [("uv", C.c_void_p), ("uvt", C.c_void_p), ("ut", C.c_void_p), ("vt", C.c_void_p),
                ("mlp", C.c_void_p)]


_P, _U32, _I, _F = C.c_void_p, C.c_uint32, C.c_int, C.c_float
_SIGS = {
    "ndgi_load": (_I, [C.POINTER(ndgi_layout), C.POINTER(ndgi_params), _I, C.POINTER(C.c_void_p)]),
    "ndgi_decode_tiles": (_I, [_P, _P, _P, _U32, _U32, _F, _P, _I, _I, _P]),
    "ndgi_decode_full": (_I, [_P, _F, _P, _I, _I, _P]),
    "ndgi_decode_full_batch": (_I, [_P, C.POINTER(_F), _U32, _P, _I, _I, _P]),
    "ndgi_decode_full_host": (_I, [_P, C.POINTER(_F), _U32, _P, _I, _I]),
    "ndgi_full_texels": (C.c_uint64, [C.POINTER(ndgi_layout)]),
    "ndgi_texel_bytes": (C.c_size_t, [_I]),
    "ndgi_device_error": (_I, [_P, C.POINTER(_U32), _I]),
    "ndgi_status_string": (C.c_char_p, [_I]),
    "ndgi_last_error": (C.c_char_p, []),
    "ndgi_free": (_I, [_P]),
    "ndgi_validate_layout": (_I, [C.POINTER(ndgi_layout), C.POINTER(_I)]),
    "ndgi_debug_bc7_decode": (_I, [_P, _U32, _U32, _P, _P]),
    "ndgi_debug_bc7_decode_hw": (_I, [_P, _U32, _U32, _P]),
    "ndgi_debug_gelu_rate": (_I, [_U32, _U32, _I, C.POINTER(_F), C.POINTER(C.c_double)]),
    "ndgi_debug_gelu_split": (_I, [_U32, C.POINTER(_U32), C.POINTER(_I)]),
    "ndgi_debug_mma_latency": (_I, [_U32, C.POINTER(C.c_double)]),
    "ndgi_debug_null_launch": (_I, [_P]),
    "ndgi_debug_launch_probe": (_I, [_I, _P]),
    "ndgi_debug_tmem_f16_probe": (_I, [_P]),
    "ndgi_debug_f16d_probe": (_I, [_U32, _U32, _U32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ndgi_vt_create": (_I, [_U32, _U32, _U32, C.POINTER(C.c_void_p)]),
    "ndgi_vt_free": (_I, [_P]),
    "ndgi_vt_request": (_I, [_P, _P, _U32, _F, _P, _P, C.POINTER(_U32), C.POINTER(_F), C.POINTER(C.c_int32)]),
    "ndgi_vt_bucket": (_I, [_P, _F, C.POINTER(C.c_int32), C.POINTER(_F)]),
    "ndgi_vt_page_table": (_I, [_P, _P]),
    "ndgi_vt_upload": (_I, [_P, _P, _P]),
    "ndgi_vt_stats": (_I, [_P, _P]),
    "ndgi_bc7_encode_mode6": (_I, [_P, _U32, _U32, _P, _P]),
    "ndgi_bc7_encode_multi": (_I, [_P, _U32, _U32, _P, _P]),
    "ndgi_train_create": (_I, [_P, C.POINTER(C.c_void_p)]),
    "ndgi_train_step": (_I, [_P, _P, _U32, _P, _P, _U32, _F, _P, _P]),
    "ndgi_train_weights": (_I, [_P, _P, _P]),
    "ndgi_train_last_grad": (_I, [_P, _P, _U32, _P]),
    "ndgi_train_export_f16": (_I, [_P, _P, _P]),
    "ndgi_train_free": (_I, [_P]),
    "ndgi_train_full_params": (C.c_size_t, [C.POINTER(ndgi_layout)]),
    "ndgi_train_full_create": (_I, [_P, _P, C.POINTER(C.c_void_p)]),
    "ndgi_train_full_export": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "ndgi_train_full_step": (_I, [_P, _P, _U32, _P, _P, _P, _U32, _F, _P, _P]),
    "ndgi_sample_lighting": (_I, [_P, _P, C.c_int32, _P, _U32, _P, _P, _U32, _F, C.POINTER(ndgi_hdr), _P, _P]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class NdgiError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.ndgi_status_string(status).decode()
        detail = _lib.ndgi_last_error().decode()
        super().__init__(f"{where}: {msg}" + (f" ({detail})" if detail else ""))


def _check(status: int, where: str) -> None:
    if status != OK:
        raise NdgiError(status, where)


def make_layout(lay: dict) -> ndgi_layout:
    """dict (ndgi_synth.layout keys) -> ndgi_layout."""
    return ndgi_layout(
        ABI_VERSION, lay["num_tiles"], lay["atlases"], lay["tiles_x"], lay["tiles_y"], lay["core"],
        lay["border"], lay["uv_res"], lay["uvt_res"], lay["uvt_depth"], lay["line_res"], lay["line_t"],
        lay["hidden"], FMT[lay["fmt_uv"]], FMT[lay["fmt_uvt"]], FMT[lay["fmt_line"]], GELU[lay["gelu"]],
        BORDER[lay["border_mode"]])


def ndgi_validate_layout(lay) -> tuple[int, bool]:
    L = lay if isinstance(lay, ndgi_layout) else make_layout(lay)
    fast = C.c_int(0)
    st = _lib.ndgi_validate_layout(C.byref(L), C.byref(fast))
    return st, bool(fast.value)


def _stream_ptr(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class Context:
    """An ndgi_ctx plus references to the (borrowed) Theta tensors."""

    def __init__(self, handle: C.c_void_p, lay: dict, theta: dict, device: int):
        self.handle = handle
        self.lay = dict(lay)
        self.theta = theta      # keeps the borrowed device buffers alive
        self.device = device
        self.layout = make_layout(lay)

    @property
    def padded(self) -> int:
        return self.lay["core"] + 2 * self.lay["border"]

    def full_texels(self) -> int:
        return int(_lib.ndgi_full_texels(C.byref(self.layout)))

    def close(self) -> None:
        """Frees the context (idempotent); also called when the object is collected."""
        lib = _lib
        if getattr(self, "handle", None) and lib is not None:
            lib.ndgi_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter shutdown: module globals may be gone
            pass


def ndgi_load(lay: dict, theta: dict, device: int = 0) -> Context:
    """theta: dict of CUDA tensors uv, uvt, ut, vt (uint8/float16) and mlp (int16/uint16 f16 bits)."""
    for k in ("uv", "uvt", "ut", "vt", "mlp"):
        t = theta[k]
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"theta[{k!r}] must be a contiguous CUDA tensor")
    L = make_layout(lay)
    P = ndgi_params(*(theta[k].data_ptr() for k in ("uv", "uvt", "ut", "vt", "mlp")))
    h = C.c_void_p()
    _check(_lib.ndgi_load(C.byref(L), C.byref(P), int(device), C.byref(h)), "ndgi_load")
    return Context(h, lay, theta, device)


def ndgi_decode_tiles(ctx: Context, tile_ids, slots, n: int, num_slots: int, t: float, out_cache,
                      fmt: str = "rgba8", mode: str = "fast", stream=None) -> None:
    """tile_ids/slots: CUDA int32/uint32 tensors (slots may be None); out_cache: CUDA tensor."""
    st = _lib.ndgi_decode_tiles(ctx.handle, C.c_void_p(tile_ids.data_ptr()),
                                C.c_void_p(slots.data_ptr()) if slots is not None else None,
                                int(n), int(num_slots), float(t), C.c_void_p(out_cache.data_ptr()),
                                OUT[fmt], MODE[mode], _stream_ptr(stream))
    _check(st, "ndgi_decode_tiles")


class TileDecoder:
    """ndgi_decode_tiles bound to fixed buffers, as a render loop holds them (the
    frame's tile ids / slots written into the same device buffers every frame):
    the pointers, formats and stream are marshalled once, so a call passes only
    (n, t) -- the per-frame Python cost of the VT path is one ctypes call."""

    def __init__(self, ctx: Context, tile_ids, slots, num_slots: int, out_cache, fmt: str = "rgba8",
                 mode: str = "fast", stream=None):
        self._f = _lib.ndgi_decode_tiles
        self._args = (ctx.handle, C.c_void_p(tile_ids.data_ptr()),
                      C.c_void_p(slots.data_ptr()) if slots is not None else None)
        self._tail = (C.c_void_p(out_cache.data_ptr()), OUT[fmt], MODE[mode], _stream_ptr(stream))
        self._num_slots = int(num_slots)
        self._keep = (ctx, tile_ids, slots, out_cache)

    def __call__(self, n: int, t: float) -> None:
        st = self._f(*self._args, n, self._num_slots, t, *self._tail)
        if st:
            _check(st, "ndgi_decode_tiles")


def ndgi_decode_full(ctx: Context, t: float, out, fmt: str = "rgba8", mode: str = "fast", stream=None) -> None:
    st = _lib.ndgi_decode_full(ctx.handle, float(t), C.c_void_p(out.data_ptr()), OUT[fmt], MODE[mode],
                               _stream_ptr(stream))
    _check(st, "ndgi_decode_full")


def ndgi_decode_full_batch(ctx: Context, ts, out, fmt: str = "rgba8", mode: str = "fast", stream=None) -> None:
    arr = (C.c_float * len(ts))(*[float(x) for x in ts])
    st = _lib.ndgi_decode_full_batch(ctx.handle, arr, len(ts), C.c_void_p(out.data_ptr()), OUT[fmt],
                                     MODE[mode], _stream_ptr(stream))
    _check(st, "ndgi_decode_full_batch")


def ndgi_decode_full_host(ctx: Context, ts, out_host, fmt: str = "rgba8", mode: str = "fast") -> None:
    """out_host: CPU tensor (pinned for overlap) of n_t * full_texels texels."""
    arr = (C.c_float * len(ts))(*[float(x) for x in ts])
    st = _lib.ndgi_decode_full_host(ctx.handle, arr, len(ts), C.c_void_p(out_host.data_ptr()), OUT[fmt],
                                    MODE[mode])
    _check(st, "ndgi_decode_full_host")


def ndgi_device_error(ctx: Context, reset: bool = False) -> int:
    v = C.c_uint32(0)
    _check(_lib.ndgi_device_error(ctx.handle, C.byref(v), int(reset)), "ndgi_device_error")
    return int(v.value)


def ndgi_free(ctx: Context) -> None:
    if ctx.handle:
        _check(_lib.ndgi_free(ctx.handle), "ndgi_free")
        ctx.handle = None


def ndgi_status_string(status: int) -> str:
    return _lib.ndgi_status_string(status).decode()


def ndgi_debug_bc7_decode(blocks, w: int, h: int, rgba, stream=None) -> None:
    _check(_lib.ndgi_debug_bc7_decode(C.c_void_p(blocks.data_ptr()), w, h, C.c_void_p(rgba.data_ptr()),
                                      _stream_ptr(stream)), "ndgi_debug_bc7_decode")


def ndgi_debug_bc7_decode_hw(blocks, w: int, h: int, rgba) -> None:
    _check(_lib.ndgi_debug_bc7_decode_hw(C.c_void_p(blocks.data_ptr()), w, h, C.c_void_p(rgba.data_ptr())),
           "ndgi_debug_bc7_decode_hw")


def ndgi_debug_gelu_rate(iters: int = 4096, mufu_pairs: int = 16, pack_f32: bool = False) -> tuple[float, float]:
    """-> (milliseconds, activations) of the GELU microbenchmark: `mufu_pairs`
    of every 16 f16x2 pairs through MUFU, the rest on the FMA pipe; pack_f32
    adds the fp32 -> f16x2 packing of the fp32-accumulator epilogue."""
    ms, acts = C.c_float(0), C.c_double(0)
    _check(_lib.ndgi_debug_gelu_rate(iters, mufu_pairs, int(pack_f32), C.byref(ms), C.byref(acts)),
           "ndgi_debug_gelu_rate")
    return float(ms.value), float(acts.value)


def ndgi_debug_gelu_split(hidden: int) -> tuple[int, bool]:
    """-> (MUFU pairs of every 16, fp32 accumulators?) compiled into the fused kernel."""
    m, f = C.c_uint32(0), C.c_int(0)
    _check(_lib.ndgi_debug_gelu_split(hidden, C.byref(m), C.byref(f)), "ndgi_debug_gelu_split")
    return int(m.value), bool(f.value)


def ndgi_debug_null_launch(stream=None) -> None:
    """An empty kernel through the C ABI (the VT launch-latency floor)."""
    _check(_lib.ndgi_debug_null_launch(_stream_ptr(stream)), "ndgi_debug_null_launch")


def ndgi_debug_launch_probe(kind: int, stream=None) -> None:
    """Launch-cost probes (0 empty, 1 + fused param block, 2 256-CTA grid with smem, 3 TMEM alloc)."""
    _check(_lib.ndgi_debug_launch_probe(int(kind), _stream_ptr(stream)), "ndgi_debug_launch_probe")


def ndgi_debug_mma_latency(iters: int = 1000) -> float:
    """SM cycles per tcgen05 round trip (st A, barrier, MMA, commit, wait, ld D)."""
    c = C.c_double(0)
    _check(_lib.ndgi_debug_mma_latency(iters, C.byref(c)), "ndgi_debug_mma_latency")
    return float(c.value)


def raw_call(name: str, *args) -> int:
    """Direct C call for contract tests (status codes instead of exceptions)."""
    return getattr(_lib, name)(*args)


def exported_symbols() -> list[str]:
    return list(_SIGS)


def upload_theta(theta: dict, device: int = 0) -> dict:
    """numpy Theta (ndgi_synth.make_theta) -> contiguous CUDA tensors (plumbing only)."""
    import numpy as np
    import torch
    out = {}
    for k, v in theta.items():
        a = np.ascontiguousarray(v)
        if a.dtype == np.uint16:
            a = a.view(np.int16)
        out[k] = torch.from_numpy(a).to(f"cuda:{device}")
    return out


# ---------------------------------------------------------------- shading side (NEXT 1)
class VT:
    """ndgi_vt: page table + strict-LRU residency of the page cache (host side)."""

    def __init__(self, num_tiles: int, capacity: int, num_buckets: int = 96):
        h = C.c_void_p()
        _check(_lib.ndgi_vt_create(int(num_tiles), int(capacity), int(num_buckets), C.byref(h)), "ndgi_vt_create")
        self.handle, self.num_tiles, self.capacity = h, int(num_tiles), int(capacity)

    def request(self, ids, t: float):
        """ids: host sequence of tile ids -> (job_ids, job_slots, t_decode, bucket) as numpy arrays / scalars."""
        import numpy as np
        ids = np.ascontiguousarray(np.asarray(ids, np.uint32))
        n = len(ids)
        jid = np.zeros(max(n, 1), np.uint32)
        jsl = np.zeros(max(n, 1), np.uint32)
        nj, td, b = C.c_uint32(0), C.c_float(0), C.c_int32(0)
        st = _lib.ndgi_vt_request(self.handle, ids.ctypes.data_as(C.c_void_p), n, float(t),
                                  jid.ctypes.data_as(C.c_void_p), jsl.ctypes.data_as(C.c_void_p), C.byref(nj),
                                  C.byref(td), C.byref(b))
        _check(st, "ndgi_vt_request")
        return jid[:nj.value].copy(), jsl[:nj.value].copy(), td.value, b.value

    def bucket(self, t: float):
        b, td = C.c_int32(0), C.c_float(0)
        _check(_lib.ndgi_vt_bucket(self.handle, float(t), C.byref(b), C.byref(td)), "ndgi_vt_bucket")
        return b.value, td.value

    def page_table(self):
        import numpy as np
        out = np.zeros((self.num_tiles, 2), np.int32)
        _check(_lib.ndgi_vt_page_table(self.handle, out.ctypes.data_as(C.c_void_p)), "ndgi_vt_page_table")
        return out

    def upload(self, page_table_dev, stream=None) -> None:
        _check(_lib.ndgi_vt_upload(self.handle, C.c_void_p(page_table_dev.data_ptr()), _stream_ptr(stream)),
               "ndgi_vt_upload")

    def stats(self):
        import numpy as np
        out = np.zeros(4, np.uint64)
        _check(_lib.ndgi_vt_stats(self.handle, out.ctypes.data_as(C.c_void_p)), "ndgi_vt_stats")
        return dict(zip(("requests", "hits", "jobs", "evictions"), (int(x) for x in out)))

    def close(self) -> None:
        lib = _lib
        if getattr(self, "handle", None) and lib is not None:
            lib.ndgi_vt_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_hdr(gamma: float, frame_times, means):
    """-> (ndgi_hdr, keep-alive arrays); means [atlases][n_frames][3]."""
    import numpy as np
    tm = np.ascontiguousarray(np.asarray(frame_times, np.float32))
    mu = np.ascontiguousarray(np.asarray(means, np.float32))
    h = ndgi_hdr(float(gamma), len(tm), tm.ctypes.data_as(C.c_void_p), mu.ctypes.data_as(C.c_void_p))
    return h, (tm, mu)


def ndgi_sample_lighting(ctx: Context, page_table, bucket: int, cache, num_slots: int, uv, atlas, n: int, t: float,
                         hdr, out_rgb, stream=None) -> None:
    """page_table int32 [tiles][2], cache uint8 [slots][P][P][4], uv float32 [n][2], atlas uint32/int32 [n] or None,
    out_rgb float32 [n][3] -- CUDA tensors; hdr from make_hdr (or (ndgi_hdr, keep))."""
    h = hdr[0] if isinstance(hdr, tuple) else hdr
    st = _lib.ndgi_sample_lighting(ctx.handle, C.c_void_p(page_table.data_ptr()), int(bucket),
                                   C.c_void_p(cache.data_ptr()), int(num_slots), C.c_void_p(uv.data_ptr()),
                                   C.c_void_p(atlas.data_ptr()) if atlas is not None else None, int(n), float(t),
                                   C.byref(h), C.c_void_p(out_rgb.data_ptr()), _stream_ptr(stream))
    _check(st, "ndgi_sample_lighting")


# ---------------------------------------------------------------- BC7 encoder (NEXT 3)
def ndgi_bc7_encode_mode6(rgba, blocks, stream=None) -> None:
    """rgba: CUDA uint8 [h][w][4]; blocks: CUDA uint8 [h/4 * w/4][16] (or any 16-B-per-block buffer)."""
    h, w = int(rgba.shape[0]), int(rgba.shape[1])
    st = _lib.ndgi_bc7_encode_mode6(C.c_void_p(rgba.data_ptr()), w, h, C.c_void_p(blocks.data_ptr()),
                                    _stream_ptr(stream))
    _check(st, "ndgi_bc7_encode_mode6")


def ndgi_bc7_encode_multi(rgba, blocks, stream=None) -> None:
    """rgba: CUDA uint8 [h][w][4]; blocks: CUDA uint8 [h/4 * w/4][16] (or any 16-B-per-block buffer)."""
    h, w = int(rgba.shape[0]), int(rgba.shape[1])
    st = _lib.ndgi_bc7_encode_multi(C.c_void_p(rgba.data_ptr()), w, h, C.c_void_p(blocks.data_ptr()),
                                    _stream_ptr(stream))
    _check(st, "ndgi_bc7_encode_multi")


# ---------------------------------------------------------------- fine-tuning (NEXT 4)
def train_full_params(lay: dict) -> int:
    L = lay if isinstance(lay, ndgi_layout) else make_layout(lay)
    return int(_lib.ndgi_train_full_params(C.byref(L)))


class Trainer:
    """ndgi_train: fp32 parameters + Adam state of every tile -- the MLP only
    (fine-tuning, R27) or, with full_init, MLP + BC-simulated maps + line grids (R28)."""

    def __init__(self, ctx: Context, full_init=None):
        h = C.c_void_p()
        if full_init is None:
            _check(_lib.ndgi_train_create(ctx.handle, C.byref(h)), "ndgi_train_create")
            self.P = 16 * ctx.lay["hidden"] + ctx.lay["hidden"] * ctx.lay["hidden"] + 5 * ctx.lay["hidden"] + 3
        else:
            _check(_lib.ndgi_train_full_create(ctx.handle, C.c_void_p(full_init.data_ptr()), C.byref(h)),
                   "ndgi_train_full_create")
            self.P = train_full_params(ctx.lay)
        self.handle, self.ctx, self.full = h, ctx, full_init is not None

    def step(self, tile_ids, samples, targets, lr: float = 1e-3, loss=None, stream=None, noise=None) -> None:
        """tile_ids CUDA int32/uint32 [n]; samples, targets CUDA float32 [n][S][3]; loss CUDA float32 [n] or None;
        noise CUDA float32 [n][S][12] (full trainer only)."""
        n, S = int(samples.shape[0]), int(samples.shape[1])
        lo = C.c_void_p(loss.data_ptr()) if loss is not None else None
        if self.full:
            st = _lib.ndgi_train_full_step(self.handle, C.c_void_p(tile_ids.data_ptr()), n,
                                           C.c_void_p(samples.data_ptr()), C.c_void_p(targets.data_ptr()),
                                           C.c_void_p(noise.data_ptr()) if noise is not None else None, S, float(lr), lo, _stream_ptr(stream))
        else:
            st = _lib.ndgi_train_step(self.handle, C.c_void_p(tile_ids.data_ptr()), n, C.c_void_p(samples.data_ptr()),
                                      C.c_void_p(targets.data_ptr()), S, float(lr), lo, _stream_ptr(stream))
        _check(st, "ndgi_train_step")

    def last_grad(self, out, stream=None) -> None:
        """out: CUDA float32 [n][P] (n <= the last step's batch)."""
        _check(_lib.ndgi_train_last_grad(self.handle, C.c_void_p(out.data_ptr()), int(out.shape[0]),
                                         _stream_ptr(stream)), "ndgi_train_last_grad")

    def weights(self, out, stream=None) -> None:
        _check(_lib.ndgi_train_weights(self.handle, C.c_void_p(out.data_ptr()), _stream_ptr(stream)), "ndgi_train_weights")

    def export_f16(self, mlp, stream=None) -> None:
        _check(_lib.ndgi_train_export_f16(self.handle, C.c_void_p(mlp.data_ptr()), _stream_ptr(stream)),
               "ndgi_train_export_f16")

    def export_full(self, stream=None) -> dict:
        """R30 (full trainer): the deployable Theta as CUDA tensors for ndgi_load
        with fmt_uv = fmt_uvt = "bc7", fmt_line = "u8"."""
        import torch
        L = self.ctx.lay
        n, R, R3, D, U, T = L["num_tiles"], L["uv_res"], L["uvt_res"], L["uvt_depth"], L["line_res"], L["line_t"]
        h = L["hidden"]
        dev = torch.device("cuda", torch.cuda.current_device())
        out = {"uv": torch.empty((n, R // 4, R // 4, 16), dtype=torch.uint8, device=dev),
               "uvt": torch.empty((n, D, R3 // 4, R3 // 4, 16), dtype=torch.uint8, device=dev),
               "ut": torch.empty((n, T, U, 2), dtype=torch.uint8, device=dev),
               "vt": torch.empty((n, T, U, 2), dtype=torch.uint8, device=dev),
               "mlp": torch.empty((n, 16 * h + h + h * h + h + 3 * h + 3), dtype=torch.int16, device=dev)}
        _check(_lib.ndgi_train_full_export(self.handle, *(C.c_void_p(out[k].data_ptr()) for k in
                                                          ("uv", "uvt", "ut", "vt", "mlp")), _stream_ptr(stream)),
               "ndgi_train_full_export")
        return out

    def close(self) -> None:
        lib = _lib
        if getattr(self, "handle", None) and lib is not None:
            lib.ndgi_train_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ndgi_debug_f16d_probe(seed: int = 1, iters: int = 64, ctas: int = 148) -> tuple[int, int]:
    """(mismatching f16x2 pairs, pairs compared): f16-D MMA vs cvt.rn of the fp32-D MMA."""
    m, t = C.c_uint64(0), C.c_uint64(0)
    _check(_lib.ndgi_debug_f16d_probe(int(seed), int(iters), int(ctas), C.byref(m), C.byref(t)),
           "ndgi_debug_f16d_probe")
    return int(m.value), int(t.value)
