"""The C-ABI library loads without a GPU and exports every entry point that
include/cellgrid_b200.h declares (no compute calls: CPU only)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "cellgrid_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("cg_create", "cg_upload", "cg_step", "cg_download", "cg_grid_export",
                 "cg_record_export", "cg_box_ids", "cg_force_phase", "cg_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2105_00039_b200 import _native
    lib = _native.load()
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding covers the same set
    assert set(_native.EXPORTED) == set(declared_symbols())


def test_abi_version_and_no_device_behaviour():
    """Without a GPU every device entry point fails loudly (no CPU fallback)."""
    from paper_2105_00039_b200 import _native
    lib = _native.load()
    assert lib.cg_abi_version() == 6
    n = ctypes.c_int(-1)
    rc = lib.cg_device_count(ctypes.byref(n))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present: covered by the gpu tests")
    assert rc != 0 or n.value == 0
    with pytest.raises(_native.NativeUnavailable):
        _native.Context(0, np.float64)


def test_status_codes_map_to_reference_exceptions():
    from paper_2105_00039_b200 import _native
    from paper_2105_00039_b200.pool import PoolCapacityError
    for rc, exc in ((_native.CG_ERR_VALUE, ValueError),
                    (_native.CG_ERR_GRID_OVERFLOW, _native.GridOverflowError),
                    (_native.CG_ERR_STENCIL, _native.StencilTooSmallError),
                    (_native.CG_ERR_POOL_CAPACITY, PoolCapacityError),
                    (_native.CG_ERR_CUDA, _native.CudaError),
                    (_native.CG_ERR_NO_DEVICE, _native.NativeUnavailable)):
        with pytest.raises(exc):
            _native.check(rc)
    _native.check(_native.CG_OK)
