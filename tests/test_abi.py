"""Host-side contract of libndgi.so (no GPU needed): the library loads, exports
every entry point include/ndgi.h declares, and validates arguments before
touching CUDA."""
import ctypes as C
import os
import re

import pytest

import ndgi_synth as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ndgi.h")


def _lib():
    import paper_2604_12625_b200 as ndgi
    return ndgi


def test_header_symbols_exported():
    ndgi = _lib()
    decl = set(re.findall(r"\b(ndgi_[a-z0-9_]+)\s*\(", open(HEADER).read()))
    decl -= {"ndgi_ctx"}
    assert {"ndgi_load", "ndgi_decode_tiles", "ndgi_decode_full"} <= decl
    so = C.CDLL(ndgi.LIB_PATH)
    for name in sorted(decl):
        assert hasattr(so, name), name
    assert decl == set(ndgi.exported_symbols())


def test_status_strings():
    ndgi = _lib()
    assert ndgi.ndgi_status_string(0) == "NDGI_OK"
    assert ndgi.ndgi_status_string(2) == "NDGI_ERR_RANGE"


def test_validate_layout():
    ndgi = _lib()
    lay, _ = S.config("c2")
    st, fast = ndgi.ndgi_validate_layout(lay)
    assert st == ndgi.OK and fast
    st, fast = ndgi.ndgi_validate_layout(dict(lay, hidden=8))
    assert st == ndgi.OK and not fast                     # reference mode only
    st, fast = ndgi.ndgi_validate_layout(dict(lay, border_mode="eval_clamp"))
    assert st == ndgi.OK and not fast
    for bad in (dict(lay, core=126), dict(lay, border=128), dict(lay, num_tiles=5), dict(lay, hidden=0),
                dict(lay, uvt_res=30), dict(lay, uv_res=0)):
        assert ndgi.ndgi_validate_layout(bad)[0] == ndgi.ERR_ARG, bad
    L = ndgi.make_layout(lay)
    L.abi_version = 99
    assert ndgi.ndgi_validate_layout(L)[0] == ndgi.ERR_ARG
    L = ndgi.make_layout(lay)
    L.fmt_line = 0                                        # line maps cannot be BC7
    assert ndgi.ndgi_validate_layout(L)[0] == ndgi.ERR_ARG


def test_null_arguments_rejected_without_cuda():
    ndgi = _lib()
    assert ndgi.raw_call("ndgi_load", None, None, 0, None) == ndgi.ERR_ARG
    L = ndgi.make_layout(S.config("c1")[0])
    out = C.c_void_p()
    assert ndgi.raw_call("ndgi_load", C.byref(L), None, 0, C.byref(out)) == ndgi.ERR_ARG
    assert ndgi.raw_call("ndgi_decode_full", None, 0.5, None, 0, 0, None) == ndgi.ERR_ARG
    assert ndgi.raw_call("ndgi_decode_tiles", None, None, None, 1, 1, 0.5, None, 0, 0, None) == ndgi.ERR_ARG
    assert ndgi.raw_call("ndgi_free", None) == ndgi.ERR_ARG
    assert ndgi.raw_call("ndgi_texel_bytes", 0) == 4 and ndgi.raw_call("ndgi_texel_bytes", 2) == 16
    assert ndgi.raw_call("ndgi_full_texels", C.byref(L)) == 4 * 128 * 128


def test_no_fallback_when_library_missing(tmp_path, monkeypatch):
    # the binding must raise, not fall back, when libndgi.so is absent
    import importlib.util
    import shutil
    pkg = tmp_path / "paper_2604_12625_b200"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_2604_12625_b200", "__init__.py"), pkg / "__init__.py")
    spec = importlib.util.spec_from_file_location("ndgi_copy", pkg / "__init__.py")
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)
