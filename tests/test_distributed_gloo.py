"""Multi-process (gloo, CPU) tests of the slab-decomposition host logic in
paper_1309_4616_b200/distributed.py: the halo exchange, the rank-ordered
slice gather, the batched/polled series driver and the transfer ledger.

The node arithmetic is supplied by a CPU test double that restates the C
ABI's es_leja_dist_* contract with the oracle's stencil (test
infrastructure only); on a GPU box the same driver runs the CUDA backend.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1309_4616_b200.decomp import TransferLedger
from paper_1309_4616_b200.distributed import DistributedCsr, RowComm, SlabComm, drive_series, global_hash_state
from paper_1309_4616_b200.sparse import synthetic_symmetric

CHUNK = 8


class OracleSlabBackend:
    """CPU restatement of one rank's es_leja_dist_* series (test double)."""

    def __init__(self, spec: orc.StencilSpec, comm: SlabComm):
        self.spec, self.comm = spec, comm
        plane = comm.plane
        self.halo_lo = torch.zeros(plane, dtype=torch.float64) if comm.rank > 0 else None
        self.halo_hi = torch.zeros(plane, dtype=torch.float64) if comm.rank < comm.world - 1 else None

    def begin(self, v, dd, xi, alpha, shift, tol):
        self.v = torch.from_numpy(np.ascontiguousarray(v))
        self.dd, self.xi, self.alpha, self.shift, self.tol = dd, xi, alpha, shift, tol
        self.w = {0: self.v}
        self.p = None
        self.k, self.consecutive, self.done, self.converged = 0, 0, False, False
        self.term, self.pnorm = float("inf"), 0.0
        self.nslices = (self.comm.lz + CHUNK - 1) // CHUNK

    def slice_counts(self, comm):
        t = torch.tensor([self.nslices], dtype=torch.int64)
        parts = [torch.empty_like(t) for _ in range(comm.world)]
        dist.all_gather(parts, t)
        return [int(p.item()) for p in parts]

    def source(self, k):  # like es_leja_dist_source, valid after the decision too
        return self.w[min(k - 1, self.k)]

    def exchange(self, k):
        self.comm.exchange(self.source(k), self.halo_lo, self.halo_hi)

    def node(self):
        out = torch.zeros(2 * self.nslices, dtype=torch.float64)
        if self.done:
            return out
        k = self.k + 1
        c = self.comm
        beta = -self.shift - self.xi[k - 1]
        wk = orc.stencil_fused(self.spec, self.alpha, beta, self.w[k - 1].numpy(), z0=c.z_lo,
                               halo_lo=None if self.halo_lo is None else self.halo_lo.numpy(),
                               halo_hi=None if self.halo_hi is None else self.halo_hi.numpy())
        pold = self.dd[0] * self.v.numpy() if self.p is None else self.p
        self.pk = pold + self.dd[k] * wk
        self.wk = wk
        w3 = wk.reshape(c.lz, -1)
        p3 = self.pk.reshape(c.lz, -1)
        for s in range(self.nslices):
            a, b = s * CHUNK, min(c.lz, (s + 1) * CHUNK)
            out[2 * s] = float(np.sum(w3[a:b] ** 2))
            out[2 * s + 1] = float(np.sum(p3[a:b] ** 2))
        return out

    def decide(self, slices_all):
        _decide(self, slices_all)

    def poll_state(self):
        return self.done

    @staticmethod
    def state_done(token):
        return token

    def end(self):
        pass

    def fetch(self):
        return self.k, self.converged, self.p

    @staticmethod
    def matvecs_of(res):
        return res[0]


def _decide(self, slices_all):
    if self.done:
        return
    k = self.k + 1
    sw = float(slices_all[0::2].sum())
    sp = float(slices_all[1::2].sum())
    self.w[k] = torch.from_numpy(self.wk)
    self.p = self.pk
    self.k = k
    self.term = abs(self.dd[k]) * np.sqrt(sw)
    self.pnorm = np.sqrt(sp)
    stop = False
    if self.tol > 0:
        if self.term <= self.tol * self.pnorm:
            self.consecutive += 1
            if self.consecutive >= 2:
                stop, self.converged = True, True
        else:
            self.consecutive = 0
    if not stop and k >= len(self.dd) - 1:
        stop, self.converged = True, self.tol == 0
    self.done = stop


class OracleRowBackend:
    """CPU restatement of one rank's es_leja_csr_dist_* series (test double):
    the local block of a DistributedCsr, gathers from the all-gathered
    vector, per-chunk slices."""

    def __init__(self, op: DistributedCsr):
        self.op, self.comm = op, op.comm
        self.xg = torch.zeros(op.comm.padded, dtype=torch.float64)
        self.local = orc.Csr(op.n, op.row_ptr, op.col_idx, op.vals)

    def begin(self, v, dd, xi, alpha, shift, tol):
        self.v = torch.from_numpy(np.ascontiguousarray(v))
        self.dd, self.xi, self.alpha, self.shift, self.tol = dd, xi, alpha, shift, tol
        self.w = {0: self.v}
        self.p = None
        self.k, self.consecutive, self.done, self.converged = 0, 0, False, False
        self.nslices = (self.comm.n_local + CHUNK - 1) // CHUNK

    slice_counts = OracleSlabBackend.slice_counts
    source = OracleSlabBackend.source
    decide = _decide
    poll_state = OracleSlabBackend.poll_state
    state_done = staticmethod(OracleSlabBackend.state_done)
    end = OracleSlabBackend.end
    fetch = OracleSlabBackend.fetch
    matvecs_of = staticmethod(OracleSlabBackend.matvecs_of)

    def exchange(self, k):
        self.comm.exchange(self.source(k), self.xg)

    def node(self):
        out = torch.zeros(2 * self.nslices, dtype=torch.float64)
        if self.done:
            return out
        k = self.k + 1
        beta = -self.shift - self.xi[k - 1]
        acc = orc.csr_fused(self.local, self.alpha, 0.0, self.xg.numpy(), use_beta=False)
        wk = acc + beta * self.w[k - 1].numpy()  # alpha * acc + beta * x[r] (_core.pyx:257)
        pold = self.dd[0] * self.v.numpy() if self.p is None else self.p
        self.pk = pold + self.dd[k] * wk
        self.wk = wk
        for s in range(self.nslices):
            a, b = s * CHUNK, min(self.comm.n_local, (s + 1) * CHUNK)
            out[2 * s] = float(np.sum(wk[a:b] ** 2))
            out[2 * s + 1] = float(np.sum(self.pk[a:b] ** 2))
        return out


def _row_worker(rank, world, port, n, tol, batch, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = synthetic_symmetric(n, 3, seed=5)
        op = DistributedCsr(a)
        c = op.comm
        # the all-gather puts every block at its padded slot
        g = torch.arange(n, dtype=torch.float64) + 1.0
        xg = torch.zeros(c.padded, dtype=torch.float64)
        c.exchange(g[c.r_lo: c.r_hi].clone(), xg)
        pos = c.padded_index(np.arange(n))
        ok_gather = np.array_equal(xg.numpy()[pos], g.numpy())
        # the local block addresses the gathered vector like the global matrix addresses x
        k0, k1 = a.row_ptr[c.r_lo], a.row_ptr[c.r_hi]
        ok_block = np.array_equal(xg.numpy()[op.col_idx], g.numpy()[a.col_idx[k0:k1]])
        lo, hi = orc.Csr(n, a.row_ptr, a.col_idx.astype(np.int32), a.vals).gershgorin()
        it = orc.interpolant(lo, hi, "phi1", -0.5, 40)
        v = np.random.default_rng(4).standard_normal(n)
        be = OracleRowBackend(op)
        be.begin(v[c.r_lo: c.r_hi], it.dd, it.xi, 1.0 / it.gamma, it.center / it.gamma, tol)
        ledger = TransferLedger()
        k, conv, p = drive_series(be, c, len(it.dd), batch=batch, ledger=ledger)
        parts = [None] * world
        dist.all_gather_object(parts, (c.r_lo, p))
        if rank == 0:
            queue.put((ok_gather and ok_block, k, conv, [q for _, q in sorted(parts, key=lambda t: t[0])],
                       ledger.last_scalars()))
        else:
            queue.put(("ok", ok_gather and ok_block))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,tol,batch", [(2, 64, 0.0, 4), (3, 50, 1e-10, 3)])
def test_row_block_series_matches_single_matrix(world, n, tol, batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_worker, args=(r, world, port, n, tol, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    main = [r for r in results if r[0] != "ok"][0]
    others = [r for r in results if r[0] == "ok"]
    ok, k, conv, parts, last = main
    assert ok and all(o[1] for o in others)
    a = synthetic_symmetric(n, 3, seed=5)
    ac = orc.Csr(n, a.row_ptr, a.col_idx.astype(np.int32), a.vals)
    lo, hi = ac.gershgorin()
    it = orc.interpolant(lo, hi, "phi1", -0.5, 40)
    v = np.random.default_rng(4).standard_normal(n)
    ref, mv = orc.newton_csr(ac, it, v, tol)
    assert k == mv and conv
    assert np.concatenate(parts).tobytes() == ref.tobytes()  # bitwise, whatever the rank count
    assert last == (world - 1) * n  # reference ledger formula (decomp.py:323)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, tol, batch, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = dims
        comm = SlabComm(nx, ny, nz)
        # halo exchange puts the neighbours' seam planes in place
        g = np.arange(nx * ny * nz, dtype=np.float64)
        local = torch.from_numpy(g[comm.z_lo * comm.plane: comm.z_hi * comm.plane].copy())
        lo = torch.zeros(comm.plane, dtype=torch.float64) if rank > 0 else None
        hi = torch.zeros(comm.plane, dtype=torch.float64) if rank < world - 1 else None
        comm.exchange(local, lo, hi)
        ok_halo = (lo is None or np.array_equal(lo.numpy(), g[(comm.z_lo - 1) * comm.plane: comm.z_lo * comm.plane])) and \
                  (hi is None or np.array_equal(hi.numpy(), g[comm.z_hi * comm.plane: (comm.z_hi + 1) * comm.plane]))
        # the series over slabs
        spec_full = orc.StencilSpec(nx, ny, nz)
        lo_, hi_ = spec_full.gershgorin()
        it = orc.interpolant(lo_, hi_, "exp", -2e-3, 30)
        v = np.random.default_rng(9).standard_normal(nx * ny * nz)
        be = OracleSlabBackend(spec_full, comm)
        be.begin(v[comm.z_lo * comm.plane: comm.z_hi * comm.plane], it.dd, it.xi, 1.0 / it.gamma,
                 it.center / it.gamma, tol)
        ledger = TransferLedger()
        k, conv, p = drive_series(be, comm, len(it.dd), batch=batch, ledger=ledger)
        parts = [None] * world
        dist.all_gather_object(parts, (comm.z_lo, p))
        hashes = global_hash_state(nx, ny, nz, comm.z_lo, comm.z_hi, "cpu")
        hparts = [None] * world
        dist.all_gather_object(hparts, hashes.numpy())
        if rank == 0:
            queue.put((ok_halo, k, conv, [q for _, q in sorted(parts, key=lambda t: t[0])], ledger.last_scalars(),
                       (ledger.apply_count, getattr(ledger, "speculative_scalars", 0)), np.concatenate(hparts)))
        else:
            queue.put(("ok", ok_halo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,tol,batch", [(2, (12, 10, 16), 0.0, 4), (3, (10, 8, 24), 1e-8, 3)])
def test_slab_series_matches_single_domain(world, dims, tol, batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, tol, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    main = [r for r in results if r[0] != "ok"][0]
    others = [r for r in results if r[0] == "ok"]
    ok_halo, k, conv, parts, last, napplies, hashes = main
    assert ok_halo and all(o[1] for o in others)
    nx, ny, nz = dims
    spec = orc.StencilSpec(nx, ny, nz)
    lo, hi = spec.gershgorin()
    it = orc.interpolant(lo, hi, "exp", -2e-3, 30)
    v = np.random.default_rng(9).standard_normal(nx * ny * nz)
    ref, mv = orc.newton_stencil(spec, it, v, tol)
    assert k == mv and conv
    assert np.concatenate(parts).tobytes() == ref.tobytes()  # bitwise, whatever the rank count
    assert last == 2 * (world - 1) * nx * ny  # reference ledger formula (decomp.py:7-8)
    napplies, speculative = napplies
    assert napplies == k  # one ledger entry per operator apply of the series
    assert speculative % (2 * (world - 1) * nx * ny) == 0  # wasted exchanges booked apart
    # the synthetic state does not depend on the partition
    assert np.array_equal(hashes, global_hash_state(nx, ny, nz, 0, nz, "cpu").numpy())


def _domain_worker(rank, world, port, queue):
    from types import SimpleNamespace

    from paper_1309_4616_b200.distributed import allreduce_scalar, rank_consistent_pointwise
    from paper_1309_4616_b200.errors import DomainError

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = SlabComm(4, 3, 6)  # z-slabs of 4x3 planes
        op = SimpleNamespace(comm=comm)

        def g_local():  # only the last rank sees u <= 0, at local index 5
            if rank == world - 1:
                raise DomainError("local", index=5)
            return "fine"

        try:
            rank_consistent_pointwise(op, g_local)
            got = None
        except DomainError as e:
            got = e.index
        ok = rank_consistent_pointwise(op, lambda: "fine") == "fine"
        mx = allreduce_scalar(comm, float(rank + 1), dist.ReduceOp.MAX)
        queue.put((rank, got, ok, mx, comm.z_lo))
    finally:
        dist.destroy_process_group()


def test_domain_error_and_norm_are_rank_consistent():
    # every rank raises DomainError with the GLOBAL index (one rank
    # raising alone would leave its peers waiting in the next series)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_domain_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    last_z_lo = results[-1][4]
    for rank, got, ok, mx, _ in results:
        assert got == last_z_lo * 12 + 5
        assert ok and mx == float(world)
