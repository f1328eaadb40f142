"""The C-ABI library builds, loads and exports every symbol include/tcg.h
declares (CPU-only: no compute calls)."""

from __future__ import annotations

import ctypes
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "tcg.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(tcg_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2112_02052_b200 import _build

    return _build.build()


def test_header_declares_expected_surface():
    names = declared_functions()
    for n in ("tcg_sgt", "tcg_spmm", "tcg_sddmm", "tcg_csr_transpose", "tcg_segment_softmax",
              "tcg_segment_softmax_backward", "tcg_agnn_forward", "tcg_quantize_tf32",
              "tcg_last_error"):
        assert n in names


def test_library_exports_all_declared(lib_path):
    lib = ctypes.CDLL(str(lib_path))
    for n in declared_functions():
        assert hasattr(lib, n), n


def test_python_binding_covers_header(lib_path):
    from paper_2112_02052_b200 import _lib

    assert set(_lib.SIGNATURES) == set(declared_functions())
    lib = _lib.load()
    assert "sm_100a" in _lib.version()
    assert lib.tcg_sgt_workspace_bytes(1000, 5000, 16) > 0


def test_cubin_is_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib_path)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_tensor_cores(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(lib_path)],
                         capture_output=True, text=True).stdout
    assert "HMMA" in out  # mma.sync tf32 in spmm_tc / sddmm_tc


def test_validation_without_gpu(lib_path):
    """Argument errors are reported before any device work."""
    from paper_2112_02052_b200 import _lib

    lib = _lib.load()
    rc = lib.tcg_sgt(None, None, 10, 0, 0, 8, None, None, None, None, None, 0, None)
    assert rc == -1
    assert "tile shape" in lib.tcg_last_error().decode()
    t = _lib.TcgTiling(4, 4, 1, 3, 2, 2, None, None, None, None, None, None)
    rc = lib.tcg_spmm(ctypes.byref(t), None, 2, 2, None, None, None, 0, None, None, None,
                      None, 2, 0, 0, 2, 1, 0, None)
    assert rc == -1 and "window range" in lib.tcg_last_error().decode()


def _header_params():
    """name -> (return type, [parameter C types]) parsed from include/tcg.h."""
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    out = {}
    for ret, name, params in re.findall(
            r"^\s*((?:const\s+)?[a-z0-9_]+\s*\**)\s*(tcg_[a-z0-9_]+)\s*\(([^)]*)\)\s*;",
            text, flags=re.M):
        ps = [p.strip() for p in params.split(",") if p.strip() and p.strip() != "void"]
        types = [re.sub(r"\s*\b[a-z_0-9]+$", "", p) if not p.endswith("*") else p for p in ps]
        out[name] = (ret.strip(), types)
    return out


def _ctype_of(c_decl: str):
    import ctypes as C

    from paper_2112_02052_b200 import _lib

    d = c_decl.replace("const ", "").strip()
    if d.endswith("*"):
        return "char_p" if d == "char*" else "ptr"
    return {"int64_t": C.c_int64, "int32_t": C.c_int32, "int": C.c_int, "size_t": C.c_size_t,
            "tcg_tiling": _lib.TcgTiling}[d]


def test_binding_signatures_match_header():
    """Every ctypes argtype agrees with the header's parameter type, position
    by position (a pointer where the header has a pointer, int64 where it has
    int64_t, ...)."""
    import ctypes as C

    from paper_2112_02052_b200 import _lib

    decls = _header_params()
    assert set(decls) == set(_lib.SIGNATURES)
    for name, (ret, params) in decls.items():
        res, args = _lib.SIGNATURES[name]
        assert len(args) == len(params), (name, params, args)
        for i, (p, a) in enumerate(zip(params, args)):
            want = _ctype_of(p)
            if want == "ptr":
                ok = a is C.c_void_p or (hasattr(a, "_type_") and a._type_ is not None)
            else:
                ok = a is want
            assert ok, f"{name} arg {i}: header {p!r}, binding {a}"
        want_r = _ctype_of(ret)
        assert (res is C.c_char_p) if want_r == "char_p" else (res is want_r), (name, ret, res)
