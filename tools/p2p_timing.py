"""Emulated two-rank peer-memory slab series on ONE device (the test
harness's in-process ranks): series time with the halo push in the slice
kernel (ES_PEER_IN_NODE=0) vs inside the two-node pass (1).  On one GPU the
"peer" stores are local, so this measures the serialized copy phase the x2
change removes, not NVLink time.  Not part of the product."""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1309_4616_b200 as es  # noqa: E402
from test_gpu_parity import _p2p_ranks  # noqa: E402
import ctypes  # noqa: E402

from paper_1309_4616_b200 import _lib  # noqa: E402
from paper_1309_4616_b200.device import ptr  # noqa: E402


def run(op, ranks, it, v, tol, rounds, gd=None):
    """_p2p_run without the host read-back: device time of one series over all ranks."""
    lib = _lib.load()
    plane = op.grid.nx * op.grid.ny
    nz = op.grid.nz
    dd, xi = it.device_coeffs()
    vd = torch.from_numpy(v).cuda()
    for q in ranks:
        q["g"] = None if gd is None else gd[q["lo"] * plane: q["hi"] * plane].clone()
        if gd is not None:
            if q["lo"] > 0:
                q["ghalo"][:plane] = gd[(q["lo"] - 1) * plane: q["lo"] * plane]
            if q["hi"] < nz:
                q["ghalo"][plane:] = gd[q["hi"] * plane: (q["hi"] + 1) * plane]
        q["v"] = vd[q["lo"] * plane: q["hi"] * plane].clone()
        q["p"] = torch.empty_like(q["v"])
        q["desc"].base = len(ranks) * rounds
    torch.cuda.synchronize()
    ev = []
    for q in ranks:
        with torch.cuda.stream(q["stream"]):
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(lib.es_leja_p2p(ctypes.byref(q["d"]), ctypes.byref(q["desc"]), ptr(q["v"]), ptr(q["p"]),
                                       ptr(dd), ptr(xi), dd.numel(), 1.0 / it.interval.halfspan,
                                       it.interval.center / it.interval.halfspan, tol, ptr(q["g"]), ptr(q["ws"]),
                                       q["ws"].numel(), q["stream"].cuda_stream), "es_leja_p2p")
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            ev.append((e0, e1))
    passes = []
    for q in ranks:
        res = _lib.SeriesResult()
        lib.es_leja_fetch(ptr(q["ws"]), ctypes.byref(res), q["stream"].cuda_stream)
        passes.append(res.passes)
    torch.cuda.synchronize()
    t0 = min(e0.elapsed_time(ev[0][0]) for e0, _ in ev)  # relative to rank 0's start
    t1 = max(ev[0][0].elapsed_time(e1) for _, e1 in ev)
    return (t1 - t0) * 1e-3, passes[0]

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = es.Grid3D(n, n, n)
op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
bounds = [(0, n // 2), (n // 2, n)]
it = es.make_interpolant(es.gershgorin_interval(op), "phi1", -2.5e-5, 17, 1e-8)
v = np.random.default_rng(3).standard_normal(g.n)
ranks, keep = _p2p_ranks(op, bounds, two=True)
gd = torch.rand(g.n, dtype=torch.float64, device="cuda") if os.environ.get("GD") == "1" else None
rounds = 0
best = {}
for rep in range(4):
    for mode in ("0", "1"):
        os.environ["ES_PEER_IN_NODE"] = mode
        dt, passes = run(op, ranks, it, v, 0.0, rounds, gd)
        rounds += passes + 1
        best[mode] = min(best.get(mode, 1e9), dt)
print(f"{n}^3 as 2 emulated slabs, 16 nodes fixed degree: halo push in slice kernel {best['0'] * 1e3:.2f} ms, "
      f"in the pass {best['1'] * 1e3:.2f} ms")
