"""CPU oracle for the NDGI tile decode (arXiv 2604.12625) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product path (``paper_2604_12625_b200``) never imports it and shares no
code with it; see ``oracle/ndgi_oracle.c`` for the definition and the
citations of every step.

This module is a thin ctypes wrapper: argument marshalling only, all
arithmetic lives in ``ndgi_oracle.c``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ndgi_oracle.c")
# ORACLE_LIB: load another build of the same source (tests/test_oracle_sanitizers.py
# runs the pins against an ASan + UBSan build)
_LIB = os.environ.get("ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")

FMT = {"bc7": 0, "u8": 1, "f16": 2, "bc1": 3, "bc3": 4, "bc5": 5}
GELU = {"erf": 0, "tanh": 1}
BORDER = {"mirror": 0, "eval_clamp": 1}


def build(force: bool = False) -> str:
    """Compile ndgi_oracle.c to liboracle.so (plain gcc, -O2, fp-contract off)."""
    if os.environ.get("ORACLE_LIB"):
        return _LIB   # an external build (sanitizer runs), never rebuilt here
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fPIC", "-shared",
             "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


class Layout(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "num_tiles", "atlases", "tiles_x", "tiles_y", "core", "border", "uv_res", "uvt_res",
        "uvt_depth", "line_res", "line_t", "hidden", "fmt_uv", "fmt_uvt", "fmt_line", "gelu",
        "border_mode")]


class Maps(C.Structure):
    _fields_ = [("uv", C.c_void_p), ("uvt", C.c_void_p), ("ut", C.c_void_p), ("vt", C.c_void_p),
                ("mlp", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P, D, I, U32 = C.c_void_p, C.c_double, C.c_int, C.c_uint32
        sig = {
            "oracle_half_to_double": (D, [C.c_uint16]),
            "oracle_bc7_decode_block": (I, [P, P]),
            "oracle_bc7_decode_image": (None, [P, I, I, P]),
            "oracle_bc1_decode_block": (None, [P, P, I]),
            "oracle_ptq_u8": (C.c_uint8, [C.c_float]),
            "oracle_float_to_half": (C.c_uint16, [C.c_float]),
            "oracle_train_full_export": (None, [P, P, P, P, P, P, P]),
            "oracle_bc4_decode_block": (None, [P, P]),
            "oracle_bc3_decode_block": (None, [P, P]),
            "oracle_bc5_decode_block": (None, [P, P]),
            "oracle_bc7_weight": (I, [I, I]),
            "oracle_bc7_subset": (I, [I, I, I]),
            "oracle_bc7_anchor": (I, [I, I, I]),
            "oracle_sample2d": (None, [P, I, I, I, I, D, D, P]),
            "oracle_sample_uvt": (None, [P, P, D, D, D, P]),
            "oracle_gamma": (None, [D, P]),
            "oracle_features": (None, [P, P, I, D, D, D, P]),
            "oracle_gelu": (D, [D, I]),
            "oracle_mlp": (None, [I, P, P, I, P]),
            "oracle_texel": (None, [P, P, I, I, I, D, P]),
            "oracle_decode_tiles": (I, [P, P, P, U32, D, P, I]),
            "oracle_decode_full": (I, [P, P, D, P, I]),
            "oracle_quantize_rgba8_f64": (None, [P, C.c_size_t, P]),
            "oracle_quantize_rgba8_f32": (None, [P, C.c_size_t, C.c_size_t, P]),
            "oracle_mlp_params": (C.c_size_t, [I]),
            "oracle_mean_at": (I, [P, P, I, D, P]),
            "oracle_bc7_encode_mode6": (None, [P, P]),
            "oracle_train_grad": (D, [P, P, I, P, P, P, I, P]),
            "oracle_train_full_params": (C.c_size_t, [P]),
            "oracle_train_full_grad": (D, [P, P, P, P, P, I, P]),
            "oracle_train_full_project": (None, [P, P]),
            "oracle_adam": (None, [P, P, P, P, I, I, D, D, D, D]),
            "oracle_bc7_encode_image_mode6": (None, [P, I, I, P]),
            "oracle_bc7_encode_multi": (I, [P, P]),
            "oracle_bc7_encode_image_multi": (None, [P, I, I, P]),
            "oracle_restore": (D, [D, D, D]),
            "oracle_sample_lighting": (I, [P, P, I, I, I, I, I, D, D, I, D, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- BC7
def bc7_decode_block(block: bytes | np.ndarray) -> tuple[np.ndarray, int]:
    """One 16-byte block -> (16x4 RGBA8 texels, bits consumed)."""
    b = np.ascontiguousarray(np.frombuffer(bytes(block), np.uint8))
    out = np.zeros(64, np.uint8)
    n = lib().oracle_bc7_decode_block(_ptr(b), _ptr(out))
    return out.reshape(16, 4), n


def bc7_decode_image(blocks: np.ndarray, w: int, h: int) -> np.ndarray:
    """Row-major BC7 blocks of a w x h image -> [h][w][4] RGBA8."""
    b = np.ascontiguousarray(blocks, dtype=np.uint8)
    out = np.zeros((h, w, 4), np.uint8)
    lib().oracle_bc7_decode_image(_ptr(b), w, h, _ptr(out))
    return out


def bcn_decode_block(fmt: str, block) -> np.ndarray:
    """R29: one BC1 / BC3 / BC4 / BC5 block -> [16][channels] uint8
    (BC1, BC3: RGBA; BC4: 1 channel; BC5: 2 channels); texel = 4*row + col."""
    b = np.frombuffer(bytes(block), np.uint8).copy()
    assert len(b) == (8 if fmt in ("bc1", "bc4") else 16)
    nch = {"bc1": 4, "bc3": 4, "bc4": 1, "bc5": 2}[fmt]
    out = np.zeros(16 * nch, np.uint8)
    if fmt == "bc1":
        lib().oracle_bc1_decode_block(_ptr(b), _ptr(out), 0)
    else:
        getattr(lib(), f"oracle_{fmt}_decode_block")(_ptr(b), _ptr(out))
    return out.reshape(16, nch)


def ptq_u8(x: float) -> int:
    return int(lib().oracle_ptq_u8(float(x)))


def float_to_half(x: float) -> int:
    return int(lib().oracle_float_to_half(float(x)))


def bc7_weight(bits: int, index: int) -> int:
    return lib().oracle_bc7_weight(bits, index)


def bc7_subset(ns: int, part: int, texel: int) -> int:
    return lib().oracle_bc7_subset(ns, part, texel)


def bc7_anchor(ns: int, part: int, subset: int) -> int:
    return lib().oracle_bc7_anchor(ns, part, subset)


# ---------------------------------------------------------------- sampling / MLP
def sample2d(data: np.ndarray, fmt: str, rx: int, ry: int, nc: int, a: float, b: float) -> np.ndarray:
    d = np.ascontiguousarray(data)
    out = np.zeros(4, np.float64)
    lib().oracle_sample2d(_ptr(d), FMT[fmt], rx, ry, nc, float(a), float(b), _ptr(out))
    return out[:nc]


def make_layout(lay: dict) -> Layout:
    return Layout(
        num_tiles=lay["num_tiles"], atlases=lay["atlases"], tiles_x=lay["tiles_x"],
        tiles_y=lay["tiles_y"], core=lay["core"], border=lay["border"], uv_res=lay["uv_res"],
        uvt_res=lay["uvt_res"], uvt_depth=lay["uvt_depth"], line_res=lay["line_res"],
        line_t=lay["line_t"], hidden=lay["hidden"], fmt_uv=FMT[lay["fmt_uv"]],
        fmt_uvt=FMT[lay["fmt_uvt"]], fmt_line=FMT[lay["fmt_line"]], gelu=GELU[lay["gelu"]],
        border_mode=BORDER[lay["border_mode"]])


class Model:
    """Holds a layout + Theta arrays (numpy, host) and calls the C oracle."""

    def __init__(self, lay: dict, theta: dict):
        self.lay = dict(lay)
        self.L = make_layout(lay)
        self.arrs = {k: np.ascontiguousarray(theta[k]) for k in ("uv", "uvt", "ut", "vt", "mlp")}
        assert self.arrs["mlp"].dtype == np.uint16
        self.M = Maps(*(self.arrs[k].ctypes.data for k in ("uv", "uvt", "ut", "vt", "mlp")))

    @property
    def padded(self) -> int:
        return self.lay["core"] + 2 * self.lay["border"]

    def features(self, k: int, u: float, v: float, t: float) -> np.ndarray:
        x = np.zeros(16, np.float64)
        lib().oracle_features(C.byref(self.L), C.byref(self.M), k, u, v, t, _ptr(x))
        return x

    def sample_uvt(self, k: int, u: float, v: float, t: float) -> np.ndarray:
        per = self.arrs["uvt"].reshape(self.lay["num_tiles"], -1)[k]
        per = np.ascontiguousarray(per)
        out = np.zeros(4, np.float64)
        lib().oracle_sample_uvt(C.byref(self.L), _ptr(per), u, v, t, _ptr(out))
        return out

    def texel(self, k: int, x: int, y: int, t: float) -> np.ndarray:
        out = np.zeros(3, np.float64)
        lib().oracle_texel(C.byref(self.L), C.byref(self.M), k, x, y, t, _ptr(out))
        return out

    def decode_tiles(self, ids, t: float, nthreads: int = 1) -> np.ndarray:
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint32))
        P = self.padded
        out = np.zeros((len(ids), P, P, 3), np.float64)
        rc = lib().oracle_decode_tiles(C.byref(self.L), C.byref(self.M), _ptr(ids), len(ids),
                                       float(t), _ptr(out), int(nthreads))
        if rc != 0:
            raise ValueError("oracle_decode_tiles: tile id out of range")
        return out

    def train_grad(self, k: int, theta: np.ndarray, uvt: np.ndarray, target: np.ndarray):
        """R27: (loss, dloss/dtheta) of tile k's MLP (fp64 master theta) over samples uvt [S][3]."""
        theta = np.ascontiguousarray(theta, np.float64)
        uvt = np.ascontiguousarray(uvt, np.float64)
        target = np.ascontiguousarray(target, np.float64)
        g = np.zeros_like(theta)
        loss = lib().oracle_train_grad(C.byref(self.L), C.byref(self.M), int(k), _ptr(theta), _ptr(uvt), _ptr(target),
                                       len(uvt), _ptr(g))
        return loss, g

    def full_params(self) -> int:
        """R28: size of one tile's full training parameter vector."""
        return int(lib().oracle_train_full_params(C.byref(self.L)))

    def train_full_grad(self, theta: np.ndarray, uvt: np.ndarray, target: np.ndarray, noise: np.ndarray):
        """R28: (loss, gradient) of one tile's full parameter vector (BC-simulated maps, noise, MLP)."""
        theta = np.ascontiguousarray(theta, np.float64)
        g = np.zeros_like(theta)
        loss = lib().oracle_train_full_grad(C.byref(self.L), _ptr(theta), _ptr(np.ascontiguousarray(uvt, np.float64)),
                                            _ptr(np.ascontiguousarray(target, np.float64)),
                                            _ptr(np.ascontiguousarray(noise, np.float64)), len(uvt), _ptr(g))
        return loss, g

    def train_full_export(self, theta: np.ndarray) -> dict:
        """R30: fp32 parameters [num_tiles][P] -> a deployable Theta (BC7 F_uv,
        BC7 F_uvt, u8 line maps, f16 MLP) in ndgi_load's dense layouts."""
        L = self.lay
        theta = np.ascontiguousarray(theta, np.float32)
        n, R, R3, D, U, T = L["num_tiles"], L["uv_res"], L["uvt_res"], L["uvt_depth"], L["line_res"], L["line_t"]
        h = L["hidden"]
        out = {"uv": np.zeros((n, R // 4, R // 4, 16), np.uint8),
               "uvt": np.zeros((n, D, R3 // 4, R3 // 4, 16), np.uint8),
               "ut": np.zeros((n, T, U, 2), np.uint8), "vt": np.zeros((n, T, U, 2), np.uint8),
               "mlp": np.zeros((n, 16 * h + h + h * h + h + 3 * h + 3), np.uint16)}
        lib().oracle_train_full_export(C.byref(self.L), _ptr(theta), *(_ptr(out[k]) for k in ("uv", "uvt", "ut", "vt", "mlp")))
        return out

    def train_full_project(self, theta: np.ndarray) -> None:
        assert theta.dtype == np.float64 and theta.flags["C_CONTIGUOUS"]
        lib().oracle_train_full_project(C.byref(self.L), _ptr(theta))

    def decode_full(self, t: float, nthreads: int = 1) -> np.ndarray:
        L = self.lay
        C_ = L["core"]
        out = np.zeros((L["atlases"], L["tiles_y"] * C_, L["tiles_x"] * C_, 3), np.float64)
        lib().oracle_decode_full(C.byref(self.L), C.byref(self.M), float(t), _ptr(out), int(nthreads))
        return out


def gamma(t: float) -> np.ndarray:
    g = np.zeros(4, np.float64)
    lib().oracle_gamma(float(t), _ptr(g))
    return g


def gelu(z: float, variant: str = "erf") -> float:
    return lib().oracle_gelu(float(z), GELU[variant])


def mlp(h: int, w_f16bits: np.ndarray, x: np.ndarray, variant: str = "erf") -> np.ndarray:
    w = np.ascontiguousarray(w_f16bits, dtype=np.uint16)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(3, np.float64)
    lib().oracle_mlp(h, _ptr(w), _ptr(xx), GELU[variant], _ptr(y))
    return y


def mlp_params(h: int) -> int:
    return lib().oracle_mlp_params(h)


def quantize_rgba8(y3: np.ndarray) -> np.ndarray:
    """RN-even(clamp(y,0,1)*255), A=255; precision follows y's dtype (f64 or f32)."""
    if y3.dtype == np.float32:
        y = np.ascontiguousarray(y3)
        stride = y.shape[-1]
        n = y.size // stride
        out = np.zeros(y.shape[:-1] + (4,), np.uint8)
        lib().oracle_quantize_rgba8_f32(_ptr(y), stride, n, _ptr(out))
        return out
    y = np.ascontiguousarray(y3, dtype=np.float64)
    assert y.shape[-1] == 3
    n = y.size // 3
    out = np.zeros(y.shape[:-1] + (4,), np.uint8)
    lib().oracle_quantize_rgba8_f64(_ptr(y), n, _ptr(out))
    return out


# ---------------------------------------------------------------- shading side (R21-R25)
def mean_at(times, means, t: float) -> np.ndarray:
    """R22: per-channel mean at t, linear between bracketing bake times; raises outside."""
    tm = np.ascontiguousarray(times, np.float64)
    mu = np.ascontiguousarray(means, np.float64).reshape(-1, 3)
    out = np.zeros(3, np.float64)
    if lib().oracle_mean_at(_ptr(tm), _ptr(mu), len(tm), float(t), _ptr(out)):
        raise ValueError("t outside the bake times")
    return out


def restore(x: float, g: float, mu: float) -> float:
    return lib().oracle_restore(float(x), float(g), float(mu))


def sample_lighting(cache: np.ndarray, page_table: np.ndarray, core: int, border: int, tiles_x: int, tiles_y: int,
                    atlas: np.ndarray, uv: np.ndarray, bucket: int, g: float, mu: np.ndarray):
    """cache [slots][P][P][4] u8, page_table [tiles][2] int32 (slot, bucket), atlas [n], uv [n][2],
    mu [atlases][3]: returns (rgb [n][3] float64, resident [n] bool)."""
    cache = np.ascontiguousarray(cache, np.uint8)
    pt = np.ascontiguousarray(page_table, np.int32)
    mu = np.ascontiguousarray(mu, np.float64).reshape(-1, 3)
    n = len(uv)
    out = np.full((n, 3), np.nan)
    ok = np.zeros(n, bool)
    o3 = np.zeros(3, np.float64)
    L = lib()
    for i in range(n):
        a = int(atlas[i])
        r = L.oracle_sample_lighting(_ptr(cache), _ptr(pt), core, border, tiles_x, tiles_y, a, float(uv[i][0]),
                                     float(uv[i][1]), int(bucket), float(g), _ptr(mu[a]), _ptr(o3))
        if r == 0:
            out[i] = o3
            ok[i] = True
    return out, ok


# ---------------------------------------------------------------- BC7 mode-6 encoder (R26)
def bc7_encode_block_mode6(px: np.ndarray) -> np.ndarray:
    """16 RGBA8 texels (texel = 4*row + col) -> one 16-byte mode-6 block."""
    px = np.ascontiguousarray(np.asarray(px, np.uint8).reshape(64))
    out = np.zeros(16, np.uint8)
    lib().oracle_bc7_encode_mode6(_ptr(px), _ptr(out))
    return out


def bc7_encode_block_multi(px: np.ndarray) -> tuple[np.ndarray, int]:
    """R31: one 4x4 RGBA8 block ([16][4] or [4][4][4]) -> (16-byte block, chosen mode)."""
    p = np.ascontiguousarray(px, np.uint8).reshape(64)
    out = np.zeros(16, np.uint8)
    m = lib().oracle_bc7_encode_multi(_ptr(p), _ptr(out))
    return out, int(m)


def bc7_encode_image_multi(rgba: np.ndarray) -> np.ndarray:
    """R31: [h][w][4] uint8 -> [h/4][w/4][16] BC7 blocks (mode 6 / 5 / 7 search)."""
    h, w = rgba.shape[:2]
    r = np.ascontiguousarray(rgba, np.uint8)
    out = np.zeros((h // 4, w // 4, 16), np.uint8)
    lib().oracle_bc7_encode_image_multi(_ptr(r), w, h, _ptr(out))
    return out


def bc7_encode_image_mode6(rgba: np.ndarray) -> np.ndarray:
    """[h][w][4] RGBA8 (h, w multiples of 4) -> [h/4 * w/4][16] blocks, row-major."""
    rgba = np.ascontiguousarray(rgba, np.uint8)
    h, w = rgba.shape[:2]
    out = np.zeros(((h // 4) * (w // 4), 16), np.uint8)
    lib().oracle_bc7_encode_image_mode6(_ptr(rgba), w, h, _ptr(out))
    return out


def adam(theta, m, v, g, step: int, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8) -> None:
    """In place, PyTorch's Adam order with bias correction (R27)."""
    for a in (theta, m, v):
        assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    g = np.ascontiguousarray(g, np.float64)
    lib().oracle_adam(_ptr(theta), _ptr(m), _ptr(v), _ptr(g), len(theta), int(step), lr, b1, b2, eps)
