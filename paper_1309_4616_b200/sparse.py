"""CSR operator for the paper's unstructured matrices (drop-in for the
reference's sparse.py).

Host arrays describe the matrix (validated like sparse.py:47-64); a device
copy (i64 row_ptr, i32 col, f64 vals) is uploaded once per device and every
product runs in the CSR kernels behind es_csr_fused_rows / es_leja_csr, with
row sums accumulated strictly in storage order (bit-identical to the
reference's compiled core).
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np
import torch

from . import _lib, timing
from .device import Workspace, empty, is_complex_data, is_host, like_input, ptr, stream_handle, to_device, to_device_z


class CsrMatrix:
    def __init__(self, nrows: int, ncols: int, row_ptr, col_idx, vals, check: bool = True):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64 if ncols > 2**31 - 1 else np.int32)
        vals = np.asarray(vals)
        if vals.dtype not in (np.float32, np.float64, np.complex128):
            vals = vals.astype(np.complex128 if np.iscomplexobj(vals) else np.float64)
        self.vals = np.ascontiguousarray(vals)
        self._dev: dict[int, tuple] = {}
        self._ws = Workspace()
        if check:
            self._validate()

    def _validate(self):
        nnz = self.vals.shape[0]
        rp = self.row_ptr
        if rp.shape != (self.nrows + 1,):
            raise ValueError("row_ptr must have length nrows+1")
        if self.col_idx.shape != (nnz,):
            raise ValueError("col_idx and vals must have equal length")
        if rp[0] != 0 or rp[-1] != nnz:
            raise ValueError("row_ptr must start at 0 and end at nnz")
        if np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr must be nondecreasing")
        if nnz and (self.col_idx.min() < 0 or self.col_idx.max() >= self.ncols):
            raise ValueError("column index out of range")
        if nnz > 1:
            row_of = np.repeat(np.arange(self.nrows), np.diff(rp))
            same = row_of[1:] == row_of[:-1]
            if np.any(same & (np.diff(self.col_idx.astype(np.int64)) <= 0)):
                raise ValueError("column indices must be strictly increasing within a row")

    nnz = property(lambda self: int(self.vals.shape[0]))
    shape = property(lambda self: (self.nrows, self.ncols))

    @property
    def n(self) -> int:
        if self.nrows != self.ncols:
            raise ValueError("operator dimension requires a square matrix")
        return self.nrows

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, vals, sum_duplicates: bool = False):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals)
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        if len(rows) and sum_duplicates:
            dup = (np.diff(rows) == 0) & (np.diff(cols) == 0)
            if dup.any():
                group = np.concatenate([[0], np.cumsum(~dup)])
                summed = np.zeros(group[-1] + 1, dtype=vals.dtype)
                np.add.at(summed, group, vals)  # same accumulation order as the reference
                head = np.concatenate([[True], ~dup])
                rows, cols, vals = rows[head], cols[head], summed
        rp = np.zeros(nrows + 1, dtype=np.int64)
        np.add.at(rp, rows + 1, 1)
        np.cumsum(rp, out=rp)
        return cls(nrows, ncols, rp, cols, vals)

    @classmethod
    def identity(cls, n: int, dtype=np.float64):
        return cls(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n), np.ones(n, dtype=dtype))

    @classmethod
    def from_dense(cls, m):
        m = np.asarray(m)
        r, c = np.nonzero(m)
        return cls.from_coo(m.shape[0], m.shape[1], r, c, m[r, c])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols), dtype=self.vals.dtype)
        out[np.repeat(np.arange(self.nrows), np.diff(self.row_ptr)), self.col_idx] = self.vals
        return out

    def diagonal(self) -> np.ndarray:
        d = np.zeros(min(self.nrows, self.ncols), dtype=self.vals.dtype)
        r = np.repeat(np.arange(self.nrows), np.diff(self.row_ptr))
        hit = r == self.col_idx
        d[r[hit]] = self.vals[hit]
        return d

    def row_abs_sums(self) -> np.ndarray:
        if self.nnz == 0:
            return np.zeros(self.nrows)
        sums = np.add.reduceat(np.concatenate([np.abs(self.vals), [0.0]]), self.row_ptr[:-1])
        sums[self.row_ptr[1:] == self.row_ptr[:-1]] = 0.0
        return sums

    def storage_bytes(self, index_width: int = 32) -> int:
        """Bytes streamed per product: vals + col (index_width) + the int64
        row_ptr actually stored (the reference undercounts it)."""
        if index_width not in (32, 64):
            raise ValueError("index_width must be 32 or 64")
        return self.vals.itemsize * self.nnz + (index_width // 8) * self.nnz + 8 * (self.nrows + 1)

    # -- device copies -------------------------------------------------------

    @property
    def is_complex(self) -> bool:
        return bool(np.iscomplexobj(self.vals))

    def device_arrays(self):
        """(row_ptr i64, col i32, vals f64 | c128) on the current device,
        uploaded once."""
        dev = torch.cuda.current_device()
        if dev not in self._dev:
            if self.col_idx.dtype != np.int32:
                raise NotImplementedError("device CSR needs 32-bit column indices")
            # f32 values are widened exactly: the reference promotes a float32
            # matrix times a float64-typed product to float64 (sparse.py:163-174)
            vals = self.vals.astype(np.float64) if self.vals.dtype == np.float32 else self.vals
            self._dev[dev] = (torch.from_numpy(self.row_ptr).to("cuda"),
                              torch.from_numpy(self.col_idx).to("cuda"),
                              torch.from_numpy(np.ascontiguousarray(vals)).to("cuda"))
        return self._dev[dev]

    def fused_apply_flat(self, alpha, beta, x):
        return fused_spmv(self, alpha, beta, x)

    def _leja_z(self, v, p_out, dd, ddabs, xi, alpha: complex, shift, tol):
        """Complex series (complex dd / vectors, the propagate path) through
        es_leja_csr_z; v, p_out complex128, dd complex128, ddabs float64."""
        lib = _lib.load()
        rp, col, vals = self.device_arrays()
        ws = self._ws.get(lib.es_leja_csr_z_workspace_bytes(self.n))
        tm = timing.active()
        ev0 = timing.event() if tm else None
        rc = lib.es_leja_csr_z_async(self.n, ptr(rp), ptr(col), ptr(vals), int(self.is_complex), ptr(v), ptr(p_out),
                                     ptr(dd), ptr(ddabs), ptr(xi), dd.numel(), alpha.real, alpha.imag, float(shift),
                                     float(tol), ptr(ws), ws.numel(), stream_handle())
        _lib.check(rc, "es_leja_csr_z_async")
        ev1 = timing.event() if tm else None
        res = _lib.SeriesResult()
        rc = lib.es_leja_fetch(ptr(ws), ctypes.byref(res), stream_handle())
        if rc != _lib.ES_ERR_NOT_CONVERGED:
            _lib.check(rc, "es_leja_fetch")
        if tm:
            tm.add(ev0, ev1, res.matvecs, res.passes)
        return res

    def _leja(self, v, p_out, dd, xi, alpha, shift, tol, gdiag=None):
        if gdiag is not None:
            raise NotImplementedError("a Jacobian diagonal is defined for stencil operators only")
        if self.is_complex:
            raise NotImplementedError("complex matrices run the complex series (_leja_z)")
        lib = _lib.load()
        rp, col, vals = self.device_arrays()
        nbytes = lib.es_leja_csr_workspace_bytes(self.n)
        ws = self._ws.get(nbytes)
        tm = timing.active()
        ev0 = timing.event() if tm else None
        rc = lib.es_leja_csr_async(self.n, ptr(rp), ptr(col), ptr(vals), ptr(v), ptr(p_out), ptr(dd), ptr(xi),
                                   dd.numel(), float(alpha), float(shift), float(tol), ptr(ws), ws.numel(),
                                   stream_handle())
        _lib.check(rc, "es_leja_csr_async")
        ev1 = timing.event() if tm else None
        res = _lib.SeriesResult()
        rc = lib.es_leja_fetch(ptr(ws), ctypes.byref(res), stream_handle())
        if rc != _lib.ES_ERR_NOT_CONVERGED:
            _lib.check(rc, "es_leja_fetch")
        if tm:
            tm.add(ev0, ev1, res.matvecs, res.passes)
        return res

    def __repr__(self):
        return f"CsrMatrix({self.nrows}x{self.ncols}, nnz={self.nnz}, dtype={self.vals.dtype})"


def csr_storage_bytes(nrows: int, nnz: int, value_bytes: int = 8, index_width: int = 32) -> int:
    return value_bytes * nnz + (index_width // 8) * nnz + 8 * (nrows + 1)


def _product(a: CsrMatrix, alpha, beta, x, use_beta: bool, row_lo: int = 0, row_hi: Optional[int] = None,
             out=None):
    host = is_host(x)
    if is_complex_data(x) or a.is_complex or isinstance(alpha, complex) or isinstance(beta, complex):
        # the reference's complex core (_core.pyx:263-278): complex alpha/beta, real or complex vals
        xd = to_device_z(x)
        rp, col, vals = a.device_arrays()
        y = empty(a.nrows, torch.complex128) if out is None else out
        hi = a.nrows if row_hi is None else row_hi
        al, be = complex(alpha), complex(beta)
        rc = _lib.load().es_csr_fused_rows_z(row_lo, hi, ptr(rp), ptr(col), ptr(vals), int(a.is_complex), ptr(xd),
                                             ptr(y), al.real, al.imag, be.real, be.imag, int(use_beta),
                                             stream_handle())
        _lib.check(rc, "es_csr_fused_rows_z")
        return like_input(y, host)
    xd = to_device(x)
    rp, col, vals = a.device_arrays()
    y = empty(a.nrows) if out is None else out
    hi = a.nrows if row_hi is None else row_hi
    rc = _lib.load().es_csr_fused_rows(row_lo, hi, ptr(rp), ptr(col), ptr(vals), ptr(xd), ptr(y),
                                       float(alpha), float(beta), int(use_beta), stream_handle())
    _lib.check(rc, "es_csr_fused_rows")
    return like_input(y, host)


def spmv(a: CsrMatrix, x, backend: str = "auto"):
    """y = A x (row sums in storage order)."""
    if tuple(np.shape(x)) != (a.ncols,):
        raise ValueError(f"vector length {tuple(np.shape(x))} does not match ncols={a.ncols}")
    return _product(a, 1.0, 0.0, x, use_beta=False)


def fused_spmv(a: CsrMatrix, alpha, beta, x, backend: str = "auto"):
    """y = alpha A x + beta x in one pass (square matrices)."""
    if a.nrows != a.ncols:
        raise ValueError("fused apply requires a square matrix")
    if tuple(np.shape(x)) != (a.ncols,):
        raise ValueError(f"vector length {tuple(np.shape(x))} does not match n={a.ncols}")
    return _product(a, alpha, beta, x, use_beta=True)


def gershgorin_bounds_csr(a: CsrMatrix, axis: str = "real"):
    if a.nrows != a.ncols:
        raise ValueError("Gershgorin bounds require a square matrix")
    if a.nrows == 0:
        return (0.0, 0.0)
    diag = a.diagonal()
    radius = np.maximum(a.row_abs_sums() - np.abs(diag), 0.0)
    c = diag.real if axis == "real" else diag.imag
    return float(np.min(c - radius)), float(np.max(c + radius))


def synthetic_symmetric(n: int, per_row: int, seed: int = 1234, diag: float = 12.0) -> CsrMatrix:
    """Seeded symmetric test operator: per_row random
    U(-1, 0) couplings per row, mirrored to A + A^T, constant diagonal,
    duplicates summed in order of appearance -- the matrix
    CsrMatrix.from_coo(..., sum_duplicates=True) builds (sparse.py:80-99),
    assembled here with one stable key sort (n = 2^22, per_row = 6: 5.5e7
    nonzeros in seconds instead of a minute of lexsort)."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n, dtype=np.int64), per_row)
    cols = rng.integers(0, n, size=n * per_row)
    vals = -rng.random(n * per_row)
    ar = np.arange(n, dtype=np.int64)
    r_all = np.concatenate([rows, cols, ar])
    c_all = np.concatenate([cols, rows, ar])
    v_all = np.concatenate([vals, vals, np.full(n, diag)])
    key = r_all * n + c_all
    del rows, cols, vals
    # stable: equal keys keep their order of appearance, like lexsort
    key, order = torch.sort(torch.from_numpy(key), stable=True)
    key, order = key.numpy(), order.numpy()
    v_all = v_all[order]
    head = np.empty(len(key), dtype=bool)
    head[0] = True
    np.not_equal(key[1:], key[:-1], out=head[1:])
    starts = np.flatnonzero(head)
    summed = v_all[starts]
    glen = np.diff(np.append(starts, len(key)))
    for j in range(1, int(glen.max()) if len(glen) else 1):  # left to right, like np.add.at
        more = np.flatnonzero(glen > j)
        summed[more] += v_all[starts[more] + j]
    ukey = key[starts]
    urow = ukey // n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(urow, minlength=n), out=rp[1:])
    return CsrMatrix(n, n, rp, (ukey - urow * n).astype(np.int32 if n <= 2**31 - 1 else np.int64), summed,
                     check=False)
