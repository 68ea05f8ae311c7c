"""Quantum propagation psi(t) = exp(-i t H) psi0 on the device (the
reference's ``propagate`` command, cli.py:304-357, as a library call).

The Hermitian generator H is a CsrMatrix (real symmetric or complex
Hermitian, e.g. read by ``read_matrix_market``); its Gershgorin interval is
real, so the interpolant targets exp(s z) with the imaginary scale
s = -i t_end and the whole series runs complex through es_leja_csr_z, with
apply_matfunc's scale-halving rescue (exp(M) = exp(M/2)^2) on top.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from .decomp import PartitionedCsr, TransferLedger, make_partition
from .device import is_host
from .errors import ConfigError
from .matfunc import MatfuncStats, apply_matfunc, gershgorin_interval


@dataclass
class PropagationResult:
    psi: object
    stats: MatfuncStats
    norm_drift: float  # | ||psi_t|| - ||psi_0|| |


def _norm(x) -> float:
    if isinstance(x, torch.Tensor):
        return float(torch.linalg.vector_norm(x).item())
    return float(np.linalg.norm(x))


def propagate(h, t_end: float, psi0=None, tol: float = 1e-8, max_degree: int = 150, workers: int = 1,
              ledger: Optional[TransferLedger] = None) -> PropagationResult:
    """exp(-i t_end H) psi0; psi0 defaults to the uniform state 1/sqrt(n)
    (cli.py:318-321).  Host arrays in give host arrays out."""
    if t_end <= 0:
        raise ConfigError("t-end must be positive")
    if tol <= 0:
        raise ConfigError("tol must be positive")
    if workers < 1:
        raise ConfigError("workers must be >= 1")
    if h.nrows != h.ncols:
        raise ConfigError("propagation requires a square (Hermitian) matrix")
    n = h.nrows
    if psi0 is None:
        psi0 = np.full(n, 1.0 / np.sqrt(n), dtype=np.complex128)
    elif is_host(psi0):
        psi0 = np.asarray(psi0).astype(np.complex128)
        if psi0.shape != (n,):
            raise ConfigError(f"state length {psi0.shape[0]} does not match matrix n={n}")
    interval = gershgorin_interval(h)
    op = h
    if workers > 1:
        op = PartitionedCsr(h, make_partition(h, workers), ledger if ledger is not None else TransferLedger())
    psi, stats = apply_matfunc(op, psi0, "exp", scale=-1j * t_end, interval=interval, tol=tol,
                               max_degree=max_degree)
    return PropagationResult(psi, stats, abs(_norm(psi) - _norm(psi0)))
