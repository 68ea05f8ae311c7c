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

The CSR operator shards as row blocks (``DistributedCsr``): per node the
ranks' w_{k-1} slices are all-gathered over NCCL into one gathered vector
(the reference's private full copy of x per worker, decomp.py:304-333;
(m-1) n scalars per node), the local rows' fused pass gathers from it, and
the same rank-ordered slice gather drives the identical stopping test.

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
        neighbours' into the halo buffers (one batched NCCL group; staged
        through host memory on a gloo group, which cannot send device
        tensors)."""
        if src.is_cuda and dist.get_backend(self.group) != "nccl":
            hl = None if halo_lo is None else torch.empty(halo_lo.shape, dtype=halo_lo.dtype)
            hh = None if halo_hi is None else torch.empty(halo_hi.shape, dtype=halo_hi.dtype)
            self.exchange(src.cpu(), hl, hh)
            if hl is not None:
                halo_lo.copy_(hl)
            if hh is not None:
                halo_hi.copy_(hh)
            return
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
        if t.is_cuda and dist.get_backend(self.group) != "nccl":  # gloo: through host memory
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
            return t
        dist.all_reduce(t, op=op, group=self.group)
        return t

    def ledger_scalars(self) -> int:
        return 2 * (self.world - 1) * self.plane


class RowComm:
    """Vector all-gather and slice gathering for one rank's row block.

    Row blocks follow make_partition (first `rem` ranks one row larger,
    decomp.py:58-83).  The gathered vector has one slot of `width` =
    max(block) doubles per rank, so the exchange is one
    ncclAllGather (all_gather_into_tensor); column indices are remapped
    into that padded layout once, when the local block is built (no padding
    when m divides n, e.g. n = 2^22 at m = 1/2/4/8)."""

    def __init__(self, n: int, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n_total = int(n)
        self.partition = make_partition(self.n_total, self.world, mode="csr_rows")
        rng = self.partition.ranges()
        self.r_lo, self.r_hi = rng[self.rank]
        self.counts = [hi - lo for lo, hi in rng]
        self.starts = np.array([lo for lo, _ in rng], dtype=np.int64)
        self.width = max(self.counts)
        self.padded = self.width * self.world
        self.n_local = self.r_hi - self.r_lo

    def padded_index(self, cols: np.ndarray) -> np.ndarray:
        """Global column index -> position in the gathered vector."""
        cols = np.asarray(cols, dtype=np.int64)
        owner = np.searchsorted(self.starts, cols, side="right") - 1
        return owner * self.width + (cols - self.starts[owner])

    def exchange(self, src: torch.Tensor, xg: torch.Tensor) -> None:
        """All ranks' slices of a row-block vector into xg (rank order)."""
        if self.n_local == self.width:
            dist.all_gather_into_tensor(xg, src[: self.width], group=self.group)
        else:
            buf = torch.zeros(self.width, dtype=src.dtype, device=src.device)
            buf[: self.n_local] = src
            dist.all_gather_into_tensor(xg, buf, group=self.group)

    def gather(self, local: torch.Tensor, counts: list[int]) -> torch.Tensor:
        return SlabComm.gather(self, local, counts)

    allreduce = SlabComm.allreduce

    def ledger_scalars(self) -> int:
        # every worker receives the other blocks (decomp.py:323)
        return (self.world - 1) * self.n_total


@dataclass
class SeriesOutcome:
    matvecs: int
    converged: int
    last_term: float
    last_pnorm: float


def drive_series(backend, comm, ndd: int, batch: int = 4, ledger: Optional[TransferLedger] = None):
    """Host loop of a multi-GPU series (slab or row block): exchange -> node
    -> gather -> decide per node, batches of `batch` nodes between
    asynchronous state polls.

    Polling lags the device by up to two batches, so a few nodes may be
    enqueued after the series has stopped (they early-exit on the device but
    their exchanges still move data).  The ledger keeps the reference's
    contract -- one entry per operator apply of the series (decomp.py:86-103)
    -- and books the speculative exchanges separately
    (``ledger.speculative_scalars``)."""
    counts = backend.slice_counts(comm)
    k, pending = 0, []
    while k < ndd - 1:
        for _ in range(batch):
            if k >= ndd - 1:
                break
            k += 1
            backend.exchange(k)
            local = backend.node()
            backend.decide(comm.gather(local, counts))
        pending.append(backend.poll_state())
        if len(pending) >= 2 and backend.state_done(pending.pop(0)):
            break
    backend.end()
    res = backend.fetch()
    if ledger is not None:
        applied = min(k, backend.matvecs_of(res))
        for _ in range(applied):
            ledger.record(comm.ledger_scalars(), 8)
        ledger.speculative_scalars = getattr(ledger, "speculative_scalars", 0) + (k - applied) * comm.ledger_scalars()
    return res


class _CudaSeriesBackend:
    """Shared part of the C ABI multi-GPU series backends: the slice gather
    counts, the shared decision (es_leja_dist_decide), asynchronous polling
    of the device state, fetch."""

    SOURCE = NSLICES = NODE = END = ""

    def __init__(self, comm, ws: torch.Tensor):
        self.comm, self.ws = comm, ws
        self.lib = _lib.load()
        self._state_off = int(self.lib.es_leja_state_offset())
        self._pinned = [torch.empty(_STATE.size, dtype=torch.uint8).pin_memory() for _ in range(3)]
        self._pi = 0

    def _after_begin(self, v):
        self.v = v
        self.n = v.numel()
        ns = ctypes.c_int32()
        _lib.check(getattr(self.lib, self.NSLICES)(ptr(self.ws), ctypes.byref(ns)))
        self.nslices = ns.value
        self.slices = torch.empty(2 * self.nslices, dtype=torch.float64, device=v.device)

    def slice_counts(self, comm):
        t = torch.tensor([self.nslices], dtype=torch.int64, device=self.slices.device)
        parts = [torch.empty_like(t) for _ in range(comm.world)]
        dist.all_gather(parts, t, group=comm.group)
        return [int(p.item()) for p in parts]

    def source(self, k: int) -> torch.Tensor:
        src = ctypes.c_void_p()
        _lib.check(getattr(self.lib, self.SOURCE)(ptr(self.ws), k, ctypes.byref(src)))
        if src.value == self.v.data_ptr():
            return self.v
        off = src.value - self.ws.data_ptr()
        return self.ws[off: off + 8 * self.n].view(torch.float64)

    def node(self) -> torch.Tensor:
        _lib.check(getattr(self.lib, self.NODE)(ptr(self.ws), ptr(self.slices), stream_handle()), self.NODE)
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
        _lib.check(getattr(self.lib, self.END)(ptr(self.ws), stream_handle()), self.END)

    @staticmethod
    def matvecs_of(res) -> int:
        return int(res.matvecs)

    def fetch(self):
        res = _lib.SeriesResult()
        rc = self.lib.es_leja_fetch(ptr(self.ws), ctypes.byref(res), stream_handle())
        if rc != _lib.ES_ERR_NOT_CONVERGED:
            _lib.check(rc, "es_leja_fetch")
        return res


class CudaSlabBackend(_CudaSeriesBackend):
    """The C ABI slab series (es_leja_dist_*) on this rank's GPU."""

    SOURCE, NSLICES, NODE, END = "es_leja_dist_source", "es_leja_dist_nslices", "es_leja_dist_node", "es_leja_dist_end"

    def __init__(self, op: StencilOperator, comm: SlabComm, ws: torch.Tensor, halo_lo, halo_hi):
        super().__init__(comm, ws)
        self.op = op
        self.halo_lo, self.halo_hi = halo_lo, halo_hi

    def begin(self, d, v, p_out, dd, xi, alpha, shift, tol, gdiag):
        rc = self.lib.es_leja_dist_begin(ctypes.byref(d), ptr(v), ptr(p_out), ptr(dd), ptr(xi), dd.numel(),
                                         float(alpha), float(shift), float(tol), ptr(gdiag), ptr(self.halo_lo),
                                         ptr(self.halo_hi), ptr(self.ws), self.ws.numel(), stream_handle())
        _lib.check(rc, "es_leja_dist_begin")
        self._after_begin(v)

    def exchange(self, k: int) -> None:
        self.comm.exchange(self.source(k), self.halo_lo, self.halo_hi)


class CudaRowBackend(_CudaSeriesBackend):
    """The C ABI row-block CSR series (es_leja_csr_dist_*) on this rank's GPU."""

    SOURCE, NSLICES, NODE, END = ("es_leja_csr_dist_source", "es_leja_csr_dist_nslices", "es_leja_csr_dist_node",
                                  "es_leja_csr_dist_end")

    def __init__(self, op: "DistributedCsr", ws: torch.Tensor):
        super().__init__(op.comm, ws)
        self.op = op

    def begin(self, v, p_out, dd, xi, alpha, shift, tol):
        rp, col, vals = self.op.device_arrays()
        rc = self.lib.es_leja_csr_dist_begin(self.op.n, ptr(rp), ptr(col), ptr(vals), ptr(self.op.xg),
                                             self.op.xg.numel(), ptr(v),
                                             ptr(p_out), ptr(dd), ptr(xi), dd.numel(), float(alpha), float(shift),
                                             float(tol), ptr(self.ws), self.ws.numel(), stream_handle())
        _lib.check(rc, "es_leja_csr_dist_begin")
        self._after_begin(v)

    def exchange(self, k: int) -> None:
        self.comm.exchange(self.source(k), self.op.xg)


def _peer_or_none(make, exchange: str, group):
    """The peer-memory resources when requested / possible on EVERY rank
    (collective; 'auto' falls back to the NCCL-driven series together).

    The data path of the peer-memory series is the kernels' own peer loads /
    stores; torch.distributed only carries the set-up (IPC handles, slice
    counts, barriers).  So an explicit exchange='p2p' also runs over a gloo
    group -- the way several processes sharing ONE device exercise the
    cross-process path (CUDA IPC, system-scope arrival counters) where NCCL
    refuses duplicate devices."""
    backend = dist.get_backend(group)
    if exchange == "nccl" or (backend != "nccl" and exchange != "p2p"):
        return None
    if exchange == "auto" and dist.get_world_size(group) == 1:
        return None  # nothing to exchange: the caller runs the single-device series
    peer, err = None, None
    try:
        peer = make()
    except Exception as e:  # IPC mapping impossible on this node
        err = e
    ok = torch.tensor([0 if peer is None else 1], device=_reduce_device(group))
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)  # every rank takes the same path
    if int(ok.item()) == 0:
        if peer is not None:
            peer.close()
        if exchange == "p2p":
            raise RuntimeError(f"peer-memory exchange unavailable: {err}")
        return None
    return peer


class _PeerMemory:
    """CUDA IPC plumbing shared by the peer-memory series: publish this
    rank's buffers, map every other rank's, fetch / count rounds."""

    def _exchange(self, comm, tensors):
        """Device addresses, valid in this process, of every rank's copy of
        `tensors` (rank order)."""
        self.lib = _lib.load()
        self._opened = getattr(self, "_opened", [])
        torch.cuda.synchronize()
        mine = [self._handle(t) for t in tensors]
        everyone = [None] * comm.world
        dist.all_gather_object(everyone, mine, group=comm.group)
        out = []
        for q, hs in enumerate(everyone):
            if q == comm.rank:
                out.append(tuple(t.data_ptr() for t in tensors))
            else:
                out.append(tuple(self._open(h) for h in hs))
        return out

    def _handle(self, t: torch.Tensor):
        h = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        _lib.check(self.lib.es_ipc_handle(t.data_ptr(), h, ctypes.byref(off)), "es_ipc_handle")
        return (h.raw, int(off.value))

    def _open(self, handle):
        raw, off = handle
        p = ctypes.c_void_p()
        _lib.check(self.lib.es_ipc_open(ctypes.create_string_buffer(raw, 64), off, ctypes.byref(p)), "es_ipc_open")
        self._opened.append(p.value)
        return int(p.value)

    poisoned = False

    def fetch(self, ws):
        res = _lib.SeriesResult()
        rc = self.lib.es_leja_fetch(ptr(ws), ctypes.byref(res), stream_handle())
        if rc != _lib.ES_ERR_NOT_CONVERGED:
            _lib.check(rc, "es_leja_fetch")
        # round 0 + one per pass over the slab (a node, or two nodes sharing a
        # pass), identical on every rank
        self.rounds += int(res.passes) + 1
        return res

    def run(self, enqueue, ws):
        """Enqueue one series and fetch its result.  The arrival counters
        only stay in step across ranks while every series completes on every
        rank: after a failure here (a peer timed out, or a rank raised before
        launching) the peers' arrivals may be ahead of ``base``, and a
        following series could read halos / slices that were never written.
        So a failure poisons these resources until ``reset()`` has run
        collectively on every rank."""
        if self.poisoned:
            raise RuntimeError("peer-memory series state is out of step after a failed series; "
                               "call reset() on every rank (collective) before the next series")
        try:
            enqueue()
            return self.fetch(ws)
        except Exception:
            self.poisoned = True
            raise

    def _zero(self):
        for t in self._resettable():
            t.zero_()

    def reset(self):
        """Collective resynchronisation after a failed series: every rank
        drains its device work, then the arrival counters, slice tables and
        exchange buffers are zeroed and the round count restarts at 0."""
        torch.cuda.synchronize()
        dist.barrier(group=self.comm.group)
        self._zero()
        self.rounds = 0
        torch.cuda.synchronize()
        dist.barrier(group=self.comm.group)
        self.poisoned = False

    def close(self):
        for p in getattr(self, "_opened", []):
            self.lib.es_ipc_close(p)
        self._opened = []


class PeerSlab(_PeerMemory):
    """Peer-memory (NVLink P2P) resources of one rank's slab series
    (es_leja_p2p): double-buffered halo planes the neighbours write into,
    the rank-ordered slice table every rank writes into, the arrival
    counter; peers' buffers mapped through CUDA IPC handles exchanged over
    torch.distributed.  Construct collectively on every rank."""

    def __init__(self, op: StencilOperator, comm: SlabComm, timeout_s: float = 30.0):
        self.lib = _lib.load()
        self.comm = c = comm
        dev = torch.device("cuda", torch.cuda.current_device())
        plane = c.plane
        # two Leja nodes per pass on the slab (the single-GPU default) where the
        # C side allows it: two-plane halos, one round per pass
        self.two = (op.two_node_passes() and op.coeff_kind() != _lib.ES_COEFF_ARRAY and c.lz >= 2
                    and all(hi - lo >= 2 for lo, hi in c.partition.ranges()))
        hp = 2 if self.two else 1
        # [lo parity 0, lo parity 1, hi parity 0, hi parity 1], hp planes each
        self.halo = torch.zeros(4 * hp * plane, dtype=torch.float64, device=dev)
        self.ghalo = torch.zeros(2 * plane, dtype=torch.float64, device=dev) if self.two else None
        d, keep = op.desc(z0=c.z_lo, lz=c.lz)
        ns = ctypes.c_int32()
        _lib.check(self.lib.es_leja_stencil_nslices(ctypes.byref(d), ctypes.byref(ns)), "es_leja_stencil_nslices")
        counts = [None] * c.world
        dist.all_gather_object(counts, int(ns.value), group=c.group)
        self.slices = torch.zeros(hp * 2 * sum(counts) * 2, dtype=torch.float64, device=dev)
        self.arrive = torch.zeros(1, dtype=torch.int64, device=dev)
        ptrs = self._exchange(c, (self.halo, self.slices, self.arrive))  # per rank: (halo, slices, arrive)
        self.rank_slices = torch.tensor([p[1] for p in ptrs], dtype=torch.int64, device=dev)
        self.rank_arrive = torch.tensor([p[2] for p in ptrs], dtype=torch.int64, device=dev)
        self.rounds = 0
        x = _lib.P2PDesc()
        x.nranks, x.rank = c.world, c.rank
        x.slice_offset, x.total_slices = sum(counts[: c.rank]), sum(counts)
        base = self.halo.data_ptr()
        for par in range(2):
            if c.rank > 0:  # receive from / send to the lower neighbour
                x.halo_lo[par] = base + 8 * par * hp * plane
                x.peer_lo[par] = ptrs[c.rank - 1][0] + 8 * (2 + par) * hp * plane  # its halo_hi
            if c.rank < c.world - 1:
                x.halo_hi[par] = base + 8 * (2 + par) * hp * plane
                x.peer_hi[par] = ptrs[c.rank + 1][0] + 8 * par * hp * plane  # its halo_lo
        x.halo_planes = hp
        x.rank_slices, x.rank_arrive = self.rank_slices.data_ptr(), self.rank_arrive.data_ptr()
        x.arrive_local = self.arrive.data_ptr()
        x.timeout_ns = int(timeout_s * 1e9)
        self.desc = x
        dist.barrier(group=c.group)

    def _resettable(self):
        return [t for t in (self.halo, self.ghalo, self.slices, self.arrive) if t is not None]

    def enqueue(self, d, v, p_out, dd, xi, alpha, shift, tol, gdiag, ws):
        """Enqueue the whole series (one graph) on the current stream."""
        self.desc.base = self.comm.world * self.rounds
        c = self.comm
        self.desc.gdiag_lo = self.desc.gdiag_hi = None
        if self.two and gdiag is not None:  # the neighbours' g' boundary planes, once per series
            lo = self.ghalo[: c.plane] if c.rank > 0 else None
            hi = self.ghalo[c.plane:] if c.rank < c.world - 1 else None
            c.exchange(gdiag, lo, hi)
            self.desc.gdiag_lo = lo.data_ptr() if lo is not None else None
            self.desc.gdiag_hi = hi.data_ptr() if hi is not None else None
        rc = self.lib.es_leja_p2p(ctypes.byref(d), ctypes.byref(self.desc), ptr(v), ptr(p_out), ptr(dd), ptr(xi),
                                  dd.numel(), float(alpha), float(shift), float(tol), ptr(gdiag), ptr(ws), ws.numel(),
                                  stream_handle())
        _lib.check(rc, "es_leja_p2p")


class PeerRows(_PeerMemory):
    """Peer-memory resources of one rank's row-block CSR series
    (es_leja_csr_p2p): the gathered vector twice (by node parity), the slice
    table and the arrival counter, peers mapped through CUDA IPC.  Construct
    collectively on every rank."""

    def __init__(self, op: "DistributedCsr", timeout_s: float = 30.0):
        self.lib = _lib.load()
        self.comm = c = op.comm
        dev = torch.device("cuda", torch.cuda.current_device())
        self.xg2 = torch.zeros(2 * c.padded, dtype=torch.float64, device=dev)
        ns = ctypes.c_int32()
        _lib.check(self.lib.es_leja_csr_nslices(op.n, ctypes.byref(ns)), "es_leja_csr_nslices")
        counts = [None] * c.world
        dist.all_gather_object(counts, int(ns.value), group=c.group)
        self.slices = torch.zeros(2 * sum(counts) * 2, dtype=torch.float64, device=dev)
        self.arrive = torch.zeros(1, dtype=torch.int64, device=dev)
        ptrs = self._exchange(c, (self.xg2, self.slices, self.arrive))
        self.rank_xg = torch.tensor([p[0] for p in ptrs], dtype=torch.int64, device=dev)
        self.rank_slices = torch.tensor([p[1] for p in ptrs], dtype=torch.int64, device=dev)
        self.rank_arrive = torch.tensor([p[2] for p in ptrs], dtype=torch.int64, device=dev)
        self.rounds = 0
        x = _lib.P2PRowsDesc()
        x.nranks, x.rank = c.world, c.rank
        x.slice_offset, x.total_slices = sum(counts[: c.rank]), sum(counts)
        x.row_offset, x.npad = c.rank * c.width, c.padded
        x.xg_local[0] = self.xg2.data_ptr()
        x.xg_local[1] = self.xg2.data_ptr() + 8 * c.padded
        x.rank_xg, x.rank_slices = self.rank_xg.data_ptr(), self.rank_slices.data_ptr()
        x.rank_arrive, x.arrive_local = self.rank_arrive.data_ptr(), self.arrive.data_ptr()
        x.timeout_ns = int(timeout_s * 1e9)
        self.desc = x
        dist.barrier(group=c.group)

    def _resettable(self):
        return [self.xg2, self.slices, self.arrive]

    def enqueue(self, op, v, p_out, dd, xi, alpha, shift, tol, ws):
        self.desc.base = self.comm.world * self.rounds
        rp, col, vals = op.device_arrays()
        rc = self.lib.es_leja_csr_p2p(op.n, ptr(rp), ptr(col), ptr(vals), ctypes.byref(self.desc), ptr(v),
                                      ptr(p_out), ptr(dd), ptr(xi), dd.numel(), float(alpha), float(shift),
                                      float(tol), ptr(ws), ws.numel(), stream_handle())
        _lib.check(rc, "es_leja_csr_p2p")


class DistributedStencil:
    """One rank's z-slab of a stencil operator; same operator protocol as
    ``StencilOperator`` (``n`` is the local point count, vectors are the
    local slab, flat x fastest)."""

    def __init__(self, op: StencilOperator, group=None, ledger: Optional[TransferLedger] = None, batch: int = 4,
                 exchange: str = "auto", peer_timeout_s: float = 30.0):
        """exchange: 'p2p' -- the peer-memory series (es_leja_p2p: halo
        planes and slice sums written over NVLink by the kernels, one graph
        per series); 'nccl' -- the host-driven series (NCCL send/recv and
        all-gather per node); 'auto' -- p2p when every rank can map its
        neighbours' memory (CUDA IPC), else nccl."""
        if op.bc.kind in ("none", "function"):
            raise GridMismatchError("slab series need homogeneous Dirichlet or Neumann boundaries")
        if exchange not in ("auto", "p2p", "nccl"):
            raise ValueError(f"unknown exchange {exchange!r}")
        g = op.grid
        self.base_operator = op
        self.comm = SlabComm(g.nx, g.ny, g.nz, group)
        # a single-plane grid has one slab (make_partition refuses m > nz,
        # decomp.py:76-77): world 1 runs the plain device series
        self.whole = g.nz == 1
        self.peer = None if self.whole else _peer_or_none(lambda: PeerSlab(op, self.comm, peer_timeout_s), exchange,
                                                          group)
        # one rank and no exchange requested: the single-device series
        self.whole = self.whole or (self.peer is None and exchange == "auto" and self.comm.world == 1)
        self.exchange = "none" if self.whole else "p2p" if self.peer is not None else "nccl"
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
        if self.whole:
            return self.base_operator._leja(v, p_out, dd, xi, alpha, shift, tol, gdiag=gdiag)
        d, keep = self.desc()
        if self.peer is not None:
            tm = timing.active()
            ev0 = timing.event() if tm else None
            ws = self._workspace()
            ev1 = []

            def go():
                self.peer.enqueue(d, v, p_out, dd, xi, alpha, shift, tol, gdiag, ws)
                ev1.append(timing.event() if tm else None)

            res = self.peer.run(go, ws)
            ev1 = ev1[0]
            for _ in range(int(res.matvecs)):
                self.ledger.record(self.comm.ledger_scalars(), 8)
            if tm:
                tm.add(ev0, ev1, res.matvecs, res.passes)
            del keep
            return res
        be = CudaSlabBackend(self.base_operator, self.comm, self._workspace(), self.halo_lo, self.halo_hi)
        tm = timing.active()
        ev0 = timing.event() if tm else None
        be.begin(d, v, p_out, dd, xi, alpha, shift, tol, gdiag)
        res = drive_series(be, self.comm, dd.numel(), self.batch, self.ledger)
        if tm:
            tm.add(ev0, timing.event(), res.matvecs, res.passes)
        del keep
        return res

    def reset_peer(self) -> None:
        """Collective: resynchronise the peer-memory series after a failure."""
        if self.peer is not None:
            self.peer.reset()

    def two_node_passes(self) -> bool:
        """Whether this rank's series run two Leja nodes per HBM pass."""
        if self.whole:
            return self.base_operator.two_node_passes()
        return self.peer is not None and self.peer.two

    def halo_exchange(self, x: torch.Tensor):
        """Fill the halo planes from the neighbours' copies of x (for fused
        prologue passes that read x's neighbours)."""
        self.comm.exchange(x, self.halo_lo, self.halo_hi)
        self.ledger.record(self.comm.ledger_scalars(), 8)


class DistributedCsr:
    """One rank's row block of a square CSR operator over torch.distributed
    (the multi-process form of decomp.PartitionedCsr); same operator
    protocol, vectors are the local rows (``n`` = local row count)."""

    def __init__(self, a, group=None, ledger: Optional[TransferLedger] = None, batch: int = 4,
                 exchange: str = "auto", peer_timeout_s: float = 30.0):
        """exchange: 'p2p' (es_leja_csr_p2p: every node stores its rows into
        every rank's gathered vector over NVLink), 'nccl' (host-driven
        all-gather per node), 'auto' (p2p when CUDA IPC works on all ranks)."""
        if exchange not in ("auto", "p2p", "nccl"):
            raise ValueError(f"unknown exchange {exchange!r}")
        if a.nrows != a.ncols:
            raise ValueError("partitioned apply requires a square matrix")
        if a.vals.dtype != np.float64:
            raise NotImplementedError("device CSR supports real fp64 values")
        self.base_operator = a
        self.comm = RowComm(a.nrows, group)
        c = self.comm
        if c.padded > 2**31 - 1:
            raise NotImplementedError("device CSR needs 32-bit column indices")
        k0, k1 = int(a.row_ptr[c.r_lo]), int(a.row_ptr[c.r_hi])
        self.row_ptr = np.ascontiguousarray(a.row_ptr[c.r_lo: c.r_hi + 1] - k0)
        self.col_idx = np.ascontiguousarray(c.padded_index(a.col_idx[k0:k1]).astype(np.int32))
        self.vals = np.ascontiguousarray(a.vals[k0:k1])
        self.ledger = ledger if ledger is not None else TransferLedger()
        self.batch = batch
        self._dev = None
        self._ws = None
        self._xg = None
        self.peer = _peer_or_none(lambda: PeerRows(self, peer_timeout_s), exchange, group)
        self.whole = self.peer is None and exchange == "auto" and c.world == 1
        self.exchange = "none" if self.whole else "p2p" if self.peer is not None else "nccl"

    @property
    def n(self) -> int:
        return self.comm.n_local

    def reset_peer(self) -> None:
        """Collective: resynchronise the peer-memory series after a failure."""
        if self.peer is not None:
            self.peer.reset()

    @property
    def xg(self) -> torch.Tensor:
        if self._xg is None:
            self._xg = torch.zeros(self.comm.padded, dtype=torch.float64, device="cuda")
        return self._xg

    def device_arrays(self):
        if self._dev is None:
            self._dev = (torch.from_numpy(self.row_ptr).cuda(), torch.from_numpy(self.col_idx).cuda(),
                         torch.from_numpy(self.vals).cuda())
        return self._dev

    def local_slice(self, x_global):
        return x_global[self.comm.r_lo: self.comm.r_hi]

    def fused_apply_flat(self, alpha, beta, x: torch.Tensor) -> torch.Tensor:
        """alpha A x + beta x on the local rows: gather, then the local block
        (alpha * acc), then + beta x with the reference's rounding order."""
        if tuple(x.shape) != (self.n,):
            raise GridMismatchError(f"local vector length {tuple(x.shape)} != {self.n}")
        self.comm.exchange(x, self.xg)
        self.ledger.record(self.comm.ledger_scalars(), 8)
        rp, col, vals = self.device_arrays()
        y = torch.empty_like(x)
        lib = _lib.load()
        _lib.check(lib.es_csr_fused_rows(0, self.n, ptr(rp), ptr(col), ptr(vals), ptr(self.xg), ptr(y),
                                         float(alpha), 0.0, 0, stream_handle()), "es_csr_fused_rows")
        _lib.check(lib.es_axpy(ptr(y), ptr(x), float(beta), ptr(y), self.n, stream_handle()), "es_axpy")
        return y

    def _workspace(self):
        nbytes = int(_lib.load().es_leja_csr_workspace_bytes(self.n))
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        return self._ws

    def _leja(self, v, p_out, dd, xi, alpha, shift, tol, gdiag=None):
        if gdiag is not None:
            raise NotImplementedError("a Jacobian diagonal is defined for stencil operators only")
        if self.whole:  # one rank: the local block is the whole matrix (unpadded, global columns)
            return self.base_operator._leja(v, p_out, dd, xi, alpha, shift, tol)
        if self.peer is not None:
            tm = timing.active()
            ev0 = timing.event() if tm else None
            ws = self._workspace()
            ev1 = []

            def go():
                self.peer.enqueue(self, v, p_out, dd, xi, alpha, shift, tol, ws)
                ev1.append(timing.event() if tm else None)

            res = self.peer.run(go, ws)
            ev1 = ev1[0]
            for _ in range(int(res.matvecs)):
                self.ledger.record(self.comm.ledger_scalars(), 8)
            if tm:
                tm.add(ev0, ev1, res.matvecs, res.passes)
            return res
        be = CudaRowBackend(self, self._workspace())
        tm = timing.active()
        ev0 = timing.event() if tm else None
        be.begin(v, p_out, dd, xi, alpha, shift, tol)
        res = drive_series(be, self.comm, dd.numel(), self.batch, self.ledger)
        if tm:
            tm.add(ev0, timing.event(), res.matvecs, res.passes)
        return res


def _reduce_device(group) -> str:
    return "cuda" if dist.get_backend(group) == "nccl" else "cpu"


def allreduce_scalar(comm, value, op, dtype=torch.float64):
    """One scalar reduced over the operator's ranks (NCCL: on the device)."""
    t = torch.tensor([value], dtype=dtype, device=_reduce_device(comm.group))
    dist.all_reduce(t, op=op, group=comm.group)
    return t.item()


def global_offset(op) -> int:
    """Global flat index of this rank's first local point / row."""
    c = op.comm
    return c.r_lo if isinstance(op, DistributedCsr) else c.z_lo * c.plane


def rank_consistent_pointwise(op, fn):
    """Run a pointwise evaluation that may raise DomainError on this rank's
    part, and make the outcome the same on every rank: if any rank hit the
    domain, all ranks raise DomainError with the smallest GLOBAL index (the
    index a single-device run reports).  Without this, one rank raises while
    its peers enter the next series and wait for it forever."""
    from .errors import DomainError

    try:
        out, bad = fn(), -1
    except DomainError as e:
        out, bad = None, int(e.index if e.index is not None else 0)
    big = 2**62
    gbad = int(allreduce_scalar(op.comm, big if bad < 0 else global_offset(op) + bad, dist.ReduceOp.MIN,
                                dtype=torch.int64))
    if gbad < big:
        raise DomainError(f"combustion nonlinearity undefined at global index {gbad}", index=gbad)
    return out


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
