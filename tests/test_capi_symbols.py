"""CPU-side checks of the C ABI library: it exists, loads without a GPU,
exports every symbol include/expstencil_b200.h declares, and the Python
structure layouts match the header (no compute calls here)."""

import ctypes
import os
import re

import pytest

from paper_1309_4616_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "expstencil_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(es_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load(require_device=False)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.es_abi_version() == 2


def test_device_query_never_errors():
    lib = _lib.load(require_device=False)
    assert lib.es_device_available() in (0, 1)


def test_struct_layouts():
    # es_stencil_desc: 5 x i64 + 3 x f64 + 2 x i32 + 7 pointers
    assert ctypes.sizeof(_lib.StencilDesc) == 5 * 8 + 3 * 8 + 2 * 4 + 7 * 8
    assert ctypes.sizeof(_lib.SeriesResult) == 4 + 4 + 8 + 8 + 4 + 4


def test_bad_descriptor_rejected_without_gpu():
    lib = _lib.load(require_device=False)
    d = _lib.StencilDesc()
    d.nx, d.ny, d.lz, d.z0, d.nz_total = 0, 1, 1, 0, 1
    assert lib.es_leja_stencil_workspace_bytes(ctypes.byref(d)) == 0
    rc = lib.es_stencil_fused_slab(ctypes.byref(d), None, None, 1.0, 0.0, None, None, None)
    assert rc == _lib.ES_ERR_ARG
    assert "bad slab extents" in _lib.last_error()


def test_product_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import numpy as np

    import paper_1309_4616_b200 as es

    op = es.StencilOperator(es.Grid3D(4, 4, 4), es.BoundaryCondition.homogeneous())
    with pytest.raises(RuntimeError, match="CUDA device"):
        op.fused_apply_flat(1.0, 0.0, np.zeros(64))
