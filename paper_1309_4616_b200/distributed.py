"""Multi-GPU slab decomposition: one process per GPU over torch.distributed.

The reference splits the z planes across an in-process thread pool and copies
the seam planes into halo buffers before every apply (decomp.py:146-266,
two-phase supersteps).  Here every rank owns one slab in its own HBM:

* per Newton-Leja node the w_{k-1} boundary planes go to the neighbouring
  ranks with NCCL send/recv (``SlabComm.exchange``) -- 2 (m-1) nx ny scalars
  per node overall, the reference's ledger formula;
* the fused node kernel streams the slab with the received planes as TMA
  halos and emits per-z-chunk partial sums of ||w||^2, ||p||^2;
* the chunk partials of all ranks are all-gathered in rank (= global z)
  order and every rank runs the identical stopping test on them
  (``es_leja_dist_decide``).  With chunk boundaries aligned to global z the
  sums are bitwise those of a single-GPU run, so decisions -- and hence p --
  do not depend on the rank count (the reference's partition invariance,
  verify.py:90-125).

The host loop enqueues nodes in batches and polls the device state with an
asynchronous copy, so no rank waits on a per-node host sync; all ranks see
the same state at the same batch boundary, which keeps their collectives in
lockstep.  The loop is backend-agnostic: the CUDA backend below drives the
C ABI; tests drive it with a CPU oracle backend over gloo.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, timing
from .decomp import TransferLedger, make_partition
from .device import ptr, stream_handle
from .errors import GridMismatchError
from .stencil import StencilOperator

_STATE = struct.Struct("<iiiidd")  # SeriesState: k, consecutive, done, converged, last_term, last_pnorm


class SlabComm:
    """Halo exchange and slice gathering for one rank's z-slab."""

    def __init__(self, nx: int, ny: int, nz: int, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nx, self.ny, self.nz = nx, ny, nz
        self.partition = make_partition(nz, self.world, mode="stencil_slab")
        self.z_lo, self.z_hi = self.partition.ranges()[self.rank]
        self.lz = self.z_hi - self.z_lo
        self.plane = nx * ny

    def _peer(self, r):
        return r if self.group is None else dist.get_global_rank(self.group, r)

    def exchange(self, src: torch.Tensor, halo_lo: Optional[torch.Tensor], halo_hi: Optional[torch.Tensor]) -> None:
        """Send this slab's first / last plane down / up; receive the
        neighbours' into the halo buffers (one batched NCCL group)."""
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, src[: self.plane], self._peer(self.rank - 1), self.group))
            ops.append(dist.P2POp(dist.irecv, halo_lo, self._peer(self.rank - 1), self.group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, src[-self.plane:], self._peer(self.rank + 1), self.group))
            ops.append(dist.P2POp(dist.irecv, halo_hi, self._peer(self.rank + 1), self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def gather(self, local: torch.Tensor, counts: list[int]) -> torch.Tensor:
        """All ranks' slices (2 doubles each) in rank order."""
        width = 2 * max(counts)
        buf = torch.zeros(width, dtype=local.dtype, device=local.device)
        buf[: local.numel()] = local
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf, group=self.group)
        return torch.cat([p[: 2 * c] for p, c in zip(parts, counts)])

    def allreduce(self, t: torch.Tensor, op) -> torch.Tensor:
        dist.all_reduce(t, op=op, group=self.group)
        return t

    def ledger_scalars(self) -> int:
        return 2 * (self.world - 1) * self.plane


@dataclass
class SeriesOutcome:
    matvecs: int
    converged: int
    last_term: float
    last_pnorm: float


def drive_series(backend, comm: SlabComm, ndd: int, batch: int = 4, ledger: Optional[TransferLedger] = None):
    """Host loop of a slab series: exchange -> node -> gather -> decide per
    node, batches of `batch` nodes between asynchronous state polls."""
    counts = backend.slice_counts(comm)
    k, pending = 0, []
    while k < ndd - 1:
        for _ in range(batch):
            if k >= ndd - 1:
                break
            k += 1
            comm.exchange(backend.source(k), backend.halo_lo, backend.halo_hi)
            if ledger is not None:
                ledger.record(comm.ledger_scalars(), 8)
            local = backend.node()
            backend.decide(comm.gather(local, counts))
        pending.append(backend.poll_state())
        if len(pending) >= 2 and backend.state_done(pending.pop(0)):
            break
    backend.end()
    return backend.fetch()


class CudaSlabBackend:
    """The C ABI slab series (es_leja_dist_*) on this rank's GPU."""

    def __init__(self, op: StencilOperator, comm: SlabComm, ws: torch.Tensor, halo_lo, halo_hi):
        self.op, self.comm, self.ws = op, comm, ws
        self.halo_lo, self.halo_hi = halo_lo, halo_hi
        self.lib = _lib.load()
        self._state_off = int(self.lib.es_leja_state_offset())
        self._pinned = [torch.empty(_STATE.size, dtype=torch.uint8).pin_memory() for _ in range(3)]
        self._pi = 0

    def begin(self, d, v, p_out, dd, xi, alpha, shift, tol, gdiag):
        self.v = v
        self.n = v.numel()
        rc = self.lib.es_leja_dist_begin(ctypes.byref(d), ptr(v), ptr(p_out), ptr(dd), ptr(xi), dd.numel(),
                                         float(alpha), float(shift), float(tol), ptr(gdiag), ptr(self.halo_lo),
                                         ptr(self.halo_hi), ptr(self.ws), self.ws.numel(), stream_handle())
        _lib.check(rc, "es_leja_dist_begin")
        ns = ctypes.c_int32()
        _lib.check(self.lib.es_leja_dist_nslices(ptr(self.ws), ctypes.byref(ns)))
        self.nslices = ns.value
        self.slices = torch.empty(2 * self.nslices, dtype=torch.float64, device=v.device)

    def slice_counts(self, comm: SlabComm):
        t = torch.tensor([self.nslices], dtype=torch.int64, device=self.slices.device)
        parts = [torch.empty_like(t) for _ in range(comm.world)]
        dist.all_gather(parts, t, group=comm.group)
        return [int(p.item()) for p in parts]

    def source(self, k: int) -> torch.Tensor:
        src = ctypes.c_void_p()
        _lib.check(self.lib.es_leja_dist_source(ptr(self.ws), k, ctypes.byref(src)))
        if src.value == self.v.data_ptr():
            return self.v
        off = src.value - self.ws.data_ptr()
        return self.ws[off: off + 8 * self.n].view(torch.float64)

    def node(self) -> torch.Tensor:
        _lib.check(self.lib.es_leja_dist_node(ptr(self.ws), ptr(self.slices), stream_handle()), "es_leja_dist_node")
        return self.slices

    def decide(self, slices_all: torch.Tensor) -> None:
        _lib.check(self.lib.es_leja_dist_decide(ptr(self.ws), ptr(slices_all), slices_all.numel() // 2,
                                                stream_handle()), "es_leja_dist_decide")

    def poll_state(self):
        buf = self._pinned[self._pi]
        self._pi = (self._pi + 1) % len(self._pinned)
        buf.copy_(self.ws[self._state_off: self._state_off + _STATE.size], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return ev, buf

    @staticmethod
    def state_done(token) -> bool:
        ev, buf = token
        ev.synchronize()
        return _STATE.unpack(bytes(buf.numpy()))[2] != 0

    def end(self):
        _lib.check(self.lib.es_leja_dist_end(ptr(self.ws), stream_handle()), "es_leja_dist_end")

    def fetch(self):
        res = _lib.SeriesResult()
        rc = self.lib.es_leja_fetch(ptr(self.ws), ctypes.byref(res), stream_handle())
        if rc != _lib.ES_ERR_NOT_CONVERGED:
            _lib.check(rc, "es_leja_fetch")
        return res


class DistributedStencil:
    """One rank's z-slab of a stencil operator; same operator protocol as
    ``StencilOperator`` (``n`` is the local point count, vectors are the
    local slab, flat x fastest)."""

    def __init__(self, op: StencilOperator, group=None, ledger: Optional[TransferLedger] = None, batch: int = 4):
        if op.bc.kind in ("none", "function"):
            raise GridMismatchError("slab series need homogeneous Dirichlet or Neumann boundaries")
        g = op.grid
        self.base_operator = op
        self.comm = SlabComm(g.nx, g.ny, g.nz, group)
        self.ledger = ledger if ledger is not None else TransferLedger()
        self.batch = batch
        dev = torch.device("cuda", torch.cuda.current_device())
        self.halo_lo = torch.zeros(g.nx * g.ny, dtype=torch.float64, device=dev) if self.comm.rank > 0 else None
        self.halo_hi = (torch.zeros(g.nx * g.ny, dtype=torch.float64, device=dev)
                        if self.comm.rank < self.comm.world - 1 else None)
        self._ws = None

    @property
    def n(self) -> int:
        return self.comm.lz * self.comm.plane

    @property
    def grid(self):
        return self.base_operator.grid

    def desc(self):
        return self.base_operator.desc(z0=self.comm.z_lo, lz=self.comm.lz)

    def local_slice(self, x_global):
        """This rank's part of a global flat vector."""
        c = self.comm
        return x_global[c.z_lo * c.plane: c.z_hi * c.plane]

    def fused_apply_flat(self, alpha, beta, x: torch.Tensor) -> torch.Tensor:
        if tuple(x.shape) != (self.n,):
            raise GridMismatchError(f"local vector length {tuple(x.shape)} != {self.n}")
        self.comm.exchange(x, self.halo_lo, self.halo_hi)
        self.ledger.record(self.comm.ledger_scalars(), 8)
        d, keep = self.desc()
        out = torch.empty_like(x)
        rc = _lib.load().es_stencil_fused_slab(ctypes.byref(d), ptr(x), ptr(out), float(alpha), float(beta),
                                               ptr(self.halo_lo), ptr(self.halo_hi), stream_handle())
        _lib.check(rc, "es_stencil_fused_slab")
        del keep
        return out

    def _workspace(self):
        d, _ = self.desc()
        nbytes = int(_lib.load().es_leja_stencil_workspace_bytes(ctypes.byref(d)))
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        return self._ws

    def _leja(self, v, p_out, dd, xi, alpha, shift, tol, gdiag=None):
        d, keep = self.desc()
        be = CudaSlabBackend(self.base_operator, self.comm, self._workspace(), self.halo_lo, self.halo_hi)
        tm = timing.active()
        ev0 = timing.event() if tm else None
        be.begin(d, v, p_out, dd, xi, alpha, shift, tol, gdiag)
        res = drive_series(be, self.comm, dd.numel(), self.batch, self.ledger)
        if tm:
            tm.add(ev0, timing.event(), res.matvecs)
        del keep
        return res

    def halo_exchange(self, x: torch.Tensor):
        """Fill the halo planes from the neighbours' copies of x (for fused
        prologue passes that read x's neighbours)."""
        self.comm.exchange(x, self.halo_lo, self.halo_hi)
        self.ledger.record(self.comm.ledger_scalars(), 8)


def global_hash_state(nx: int, ny: int, nz: int, z_lo: int, z_hi: int, device) -> torch.Tensor:
    """Partition-independent synthetic state u0 = 1 + 0.1 * h(i), h a
    64-bit integer hash of the global index i (no host array of the full
    grid: every rank builds only its slab)."""
    plane = nx * ny
    i = torch.arange(z_lo * plane, z_hi * plane, dtype=torch.int64, device=device)
    h = i * -7046029254386353131  # 0x9E3779B97F4A7C15 as int64 (wrapping multiply)
    h = h ^ (h >> 31)
    h = (h * -4658895280553007687) & 0x7FFFFFFFFFFFFFFF  # 0xBF58476D1CE4E5B9
    h = h ^ (h >> 29)
    frac = (h & ((1 << 52) - 1)).to(torch.float64) / float(1 << 52)
    return 1.0 + 0.1 * frac
