"""The peer-memory multi-GPU series across REAL processes.

One process per rank, as on an 8-GPU box, except that the ranks here share
the one visible B200 (the sandbox and the driver's GPU tiers expose one
device).  Everything the cross-process path depends on is exercised: CUDA
IPC handles exported in one process and mapped in another
(``es_ipc_handle`` / ``es_ipc_open``), peer stores of halo planes / vector
slices into another process's buffers, system-scope arrival counters and
spin barriers across contexts (time-sliced on one device), the rank-ordered
slice tables, the shared stopping decision.  torch.distributed runs on gloo
here -- NCCL refuses two ranks on one device -- and only carries the set-up;
the series' data path is the kernels' own.

Checked: bitwise equality with the single-domain series (matvec counts
included) for slab series (one- and two-node passes) and CSR row blocks, an
exponential Rosenbrock step and an exp-Euler trajectory with the observer's
global norm, and the failure protocol -- a rank that never launches makes
its peer time out, both sides are poisoned, ``reset_peer()`` (collective)
resynchronises and the next series is bitwise again.
"""

import os
import socket
import traceback

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

import paper_1309_4616_b200 as es  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stencil_case():
    g = es.Grid3D(64, 40, 64)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    v = np.random.default_rng(21).standard_normal(g.n)
    return g, op, v


def _csr_case():
    a = es.synthetic_symmetric(40_000, 6, seed=22)
    v = np.random.default_rng(23).standard_normal(a.nrows)
    return a, v


def _worker(rank, world, port, which, queue):
    import torch.distributed as dist

    from paper_1309_4616_b200.distributed import DistributedCsr, DistributedStencil

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CUDA_DEVICE_MAX_CONNECTIONS="32")
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = {}
        if which in ("slab", "slab_one", "failure"):
            if which == "slab_one":
                os.environ["ES_TB"] = "0"
            g, op, v = _stencil_case()
            dop = DistributedStencil(op, exchange="p2p", peer_timeout_s=4.0)
            out["exchange"], out["two"] = dop.exchange, dop.two_node_passes()
            it = es.make_interpolant(es.gershgorin_interval(op), "exp", -2e-4, 150, 1e-10)
            vl = torch.from_numpy(np.ascontiguousarray(dop.local_slice(v))).cuda()
            if which == "failure":
                if rank == 0:  # rank 1 never launches this series: rank 0 must time out, not hang
                    try:
                        es.newton_apply(dop, it, vl, 1e-10)
                        out["timeout"] = "no error"
                    except Exception as e:  # noqa: BLE001
                        out["timeout"] = type(e).__name__ + ": " + str(e)
                    try:
                        es.newton_apply(dop, it, vl, 1e-10)
                        out["poisoned"] = "no error"
                    except RuntimeError as e:
                        out["poisoned"] = str(e)
                dist.barrier()
                dop.reset_peer()
            p, mv = es.newton_apply(dop, it, vl, 1e-10)
            p2, mv2 = es.newton_apply(dop, it, vl, 0.0)  # a second series continues the round counters
            out.update(z_lo=dop.comm.z_lo, p=p.cpu().numpy(), mv=mv, p2=p2.cpu().numpy(), mv2=mv2)
        elif which == "csr":
            a, v = _csr_case()
            dop = DistributedCsr(a, exchange="p2p", peer_timeout_s=4.0)
            out["exchange"] = dop.exchange
            it = es.make_interpolant(es.gershgorin_interval(a), "phi1", -1.0, 150, 1e-8)
            vl = torch.from_numpy(np.ascontiguousarray(dop.local_slice(v))).cuda()
            p, mv = es.newton_apply(dop, it, vl, 1e-8)
            out.update(z_lo=dop.comm.r_lo, p=p.cpu().numpy(), mv=mv)
        elif which == "steps":
            g = es.Grid3D(48, 40, 32)
            op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
            dop = DistributedStencil(op, exchange="p2p", peer_timeout_s=4.0)
            u0 = 1.0 + 0.1 * np.random.default_rng(24).random(g.n)
            ul = torch.from_numpy(np.ascontiguousarray(dop.local_slice(u0))).cuda()
            prob = es.SemilinearProblem(operator=dop, nonlinearity=es.combustion_g, u0=ul,
                                        interval=es.gershgorin_interval(op))
            ros = es.RosenbrockStepper(prob, 1e-8)
            ur, st = ros.step(ul, 0.0, 2e-4)
            obs = []
            ue = es.integrate(prob, es.StepperConfig(h=1e-4, t_end=3e-4, tol=1e-8),
                              observer=lambda k, t, mv, mx: obs.append((k, mv, mx)))
            out.update(z_lo=dop.comm.z_lo, ur=ur.cpu().numpy(), mvr=st.matvecs, ue=ue.cpu().numpy(), obs=obs)
        queue.put((rank, out))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - surfaced by the parent
        queue.put((rank, {"error": traceback.format_exc()}))


def _run(which, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, which, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert "error" not in res[r], res[r]["error"]
    for p in procs:
        assert p.exitcode == 0
    return [res[r] for r in range(world)]


@pytest.mark.parametrize("which", ["slab", "slab_one"])
def test_slab_series_two_processes_bitwise(which, monkeypatch):
    parts = _run(which)
    assert all(o["exchange"] == "p2p" for o in parts)
    assert all(o["two"] == (which == "slab") for o in parts)
    if which == "slab_one":
        monkeypatch.setenv("ES_TB", "0")
    g, op, v = _stencil_case()
    it = es.make_interpolant(es.gershgorin_interval(op), "exp", -2e-4, 150, 1e-10)
    vd = torch.from_numpy(v).cuda()
    ref, mv = es.newton_apply(op, it, vd, 1e-10)
    ref2, mv2 = es.newton_apply(op, it, vd, 0.0)
    parts.sort(key=lambda o: o["z_lo"])
    assert all(o["mv"] == mv and o["mv2"] == mv2 for o in parts)
    assert np.concatenate([o["p"] for o in parts]).tobytes() == ref.cpu().numpy().tobytes()
    assert np.concatenate([o["p2"] for o in parts]).tobytes() == ref2.cpu().numpy().tobytes()


def test_csr_row_blocks_two_processes_bitwise():
    parts = _run("csr")
    assert all(o["exchange"] == "p2p" for o in parts)
    a, v = _csr_case()
    it = es.make_interpolant(es.gershgorin_interval(a), "phi1", -1.0, 150, 1e-8)
    ref, mv = es.newton_apply(a, it, torch.from_numpy(v).cuda(), 1e-8)
    parts.sort(key=lambda o: o["z_lo"])
    assert all(o["mv"] == mv for o in parts)
    assert np.concatenate([o["p"] for o in parts]).tobytes() == ref.cpu().numpy().tobytes()


def test_steps_two_processes_match_single_device():
    parts = _run("steps")
    parts.sort(key=lambda o: o["z_lo"])
    g = es.Grid3D(48, 40, 32)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u0 = 1.0 + 0.1 * np.random.default_rng(24).random(g.n)
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=torch.from_numpy(u0).cuda())
    ur, st = es.RosenbrockStepper(prob, 1e-8).step(prob.u0, 0.0, 2e-4)
    assert all(o["mvr"] == st.matvecs for o in parts)
    got = np.concatenate([o["ur"] for o in parts])
    ref = ur.cpu().numpy()
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    obs = []
    ue = es.integrate(prob, es.StepperConfig(h=1e-4, t_end=3e-4, tol=1e-8),
                      observer=lambda k, t, mv, mx: obs.append((k, mv, mx)))
    for o in parts:  # every rank's observer sees the global max-norm and the same matvecs
        assert [(k, mv) for k, mv, _ in o["obs"]] == [(k, mv) for k, mv, _ in obs]
        np.testing.assert_allclose([mx for _, _, mx in o["obs"]], [mx for _, _, mx in obs], rtol=1e-12)
    got = np.concatenate([o["ue"] for o in parts])
    assert np.max(np.abs(got - ue.cpu().numpy())) <= 1e-12 * np.max(np.abs(ue.cpu().numpy()))


def test_missing_rank_times_out_poisons_and_resets():
    parts = _run("failure")
    assert "did not arrive" in parts[0]["timeout"], parts[0]["timeout"]
    assert "reset()" in parts[0]["poisoned"], parts[0]["poisoned"]
    g, op, v = _stencil_case()
    it = es.make_interpolant(es.gershgorin_interval(op), "exp", -2e-4, 150, 1e-10)
    ref, mv = es.newton_apply(op, it, torch.from_numpy(v).cuda(), 1e-10)
    parts.sort(key=lambda o: o["z_lo"])
    assert all(o["mv"] == mv for o in parts)
    assert np.concatenate([o["p"] for o in parts]).tobytes() == ref.cpu().numpy().tobytes()
