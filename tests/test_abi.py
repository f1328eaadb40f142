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
