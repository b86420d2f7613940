"""The C-ABI boundary: the shared library loads and exports exactly what
include/warmgray_b200.h declares, and the Python binding agrees with it.
No compute calls are made here (no GPU in the build container)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2108_13656_b200 import _lib

HEADER = os.path.join(ROOT, "include", "warmgray_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    decls = re.findall(r"WG_API\s+([\w\s\*]+?)\s*\b(wg_\w+)\s*\(([^)]*)\)\s*;", text)
    out = {}
    for ret, name, args in decls:
        args = args.strip()
        n = 0 if args in ("", "void") else len(args.split(","))
        out[name] = (ret.strip(), n)
    return out


def test_header_parses():
    fns = header_functions()
    assert len(fns) >= 30
    assert "wg_decolor_u8" in fns and "wg_host_decolor_rows_f64" in fns


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in header_functions():
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                        check=True).stdout
    exported = set(re.findall(r"\sT\s(wg_\w+)", nm))
    assert exported == set(header_functions()), exported ^ set(header_functions())


def test_binding_matches_header():
    fns = header_functions()
    assert set(_lib.SIGNATURES) == set(fns)
    for name, (ret, n) in fns.items():
        assert len(_lib.SIGNATURES[name][1]) == n, name


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_info_calls_without_gpu():
    lib = _lib.load()
    assert lib.wg_version() == 100
    assert lib.wg_device_count() >= 0
    assert lib.wg_hdr_scratch_bytes(2, 1000) >= 2 * 1000 * 4


def test_argument_errors_are_value_errors():
    lib = _lib.load()
    # parameter validation happens before any device work
    assert lib.wg_decolor_u8(None, None, 10, 0.5, 0.8, None) == -1
    with pytest.raises(ValueError, match="beta_r"):
        _lib.call("wg_decolor_u8", 1, 1, 10, 0.5, 0.8, None)
    with pytest.raises(ValueError, match="slope"):
        _lib.call("wg_sigmoid_f64", 1, 1, 10, 0.5, float("inf"), None)
    with pytest.raises(ValueError, match="size"):
        _lib.call("wg_decolor_f32", 1, 1, -1, 0.55, 0.8, None)
    with pytest.raises(ValueError, match="row range"):
        _lib.call("wg_host_decolor_rows_f64", 1, 1, 4, 4, 0.55, 0.8, 3, 5, 0)


def test_no_device_is_a_cuda_error():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.CudaError, match="no CUDA device"):
        _lib.call("wg_host_decolor_u8", 1, 1, 1, 0.55, 0.8, 0)
