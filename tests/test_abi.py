"""CPU checks of the C-ABI boundary: libgsgpc.so loads (no GPU needed) and exports every
symbol include/gsgpc.h declares; the Python binding covers the same set."""
import ctypes
import os
import subprocess

import pytest

from paper_2101_11751_b200 import _lib


def test_library_exists_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "libgsgpc.so must be built in-tree"
    L = ctypes.CDLL(_lib.LIB_PATH)
    assert L is not None


def test_exports_every_header_symbol():
    declared = _lib.header_symbols()
    assert len(declared) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_python_binding_covers_header():
    declared = set(_lib.header_symbols())
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def test_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_and_no_device_errors_cleanly():
    L = _lib.load()
    assert b"sm_100a" in L.gsgpc_version()
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    code = L.gsgpc_ctx_create(0, ctypes.byref(h))
    assert code == _lib.CUDA_ERROR  # fails loudly, no CPU fallback


def test_fit_grid_to_data_abi():
    L = _lib.load()
    import numpy as np

    lo = np.zeros(2)
    hi = np.ones(2)
    sz = np.array([80, 20], np.int64)
    g = _lib.Grid_t()
    assert L.gsgpc_fit_grid_to_data(2, lo.ctypes.data, hi.ctypes.data, sz.ctypes.data, _lib.CUBIC,
                                    ctypes.byref(g)) == 0
    s = 1.0 / (80 - 5)
    assert g.min[0] == 0.0 - 2 * s and g.max[0] == 1.0 + 2 * s and g.size[1] == 20
    sz[0] = 5
    assert L.gsgpc_fit_grid_to_data(2, lo.ctypes.data, hi.ctypes.data, sz.ctypes.data, _lib.CUBIC,
                                    ctypes.byref(g)) == _lib.INVALID_ARGUMENT
