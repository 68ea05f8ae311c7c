"""Host-side cost of one C1 exponential-Euler step through the public API
(cProfile over many steps; the device kernel is ~75 us).  Not part of the
product."""

import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1309_4616_b200 as es  # noqa: E402
from paper_1309_4616_b200.integrator import _StepWorkspace  # noqa: E402

g = es.Grid3D(256, 256, 1)
op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
u0 = 1.0 + 0.1 * np.random.default_rng(1234).random(g.n)
prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
ws = _StepWorkspace(prob, 1e-5, 1e-8, 150)
u = torch.from_numpy(u0).cuda()
for _ in range(20):
    ws.step(u, 0.0)
torch.cuda.synchronize()
n = 300
t0 = time.perf_counter()
for _ in range(n):
    ws.step(u, 0.0)
torch.cuda.synchronize()
print(f"wall per step {1e6 * (time.perf_counter() - t0) / n:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    ws.step(u, 0.0)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# the C call alone, arguments prebuilt (what remains without the Python layer)
import ctypes  # noqa: E402

from paper_1309_4616_b200 import _lib  # noqa: E402
from paper_1309_4616_b200.device import ptr, stream_handle  # noqa: E402

lib = _lib.load()
d, keep = op.desc()
nbytes = lib.es_leja_stencil_workspace_bytes(ctypes.byref(d))
ws.step(u, 0.0)
ws_exp, ws_phi = op._ws.get(nbytes), ws._ws_phi.get(nbytes)
dde, xi = ws.exp_interp.device_coeffs()
ddp, _ = ws.phi_interp.device_coeffs()
iv = ws.exp_interp.interval
out = torch.empty_like(u)
res = _lib.StepResult()
args = (ctypes.byref(d), ptr(u), ptr(out), ptr(dde), dde.numel(), ptr(ddp), ddp.numel(), ptr(xi), 1.0 / iv.halfspan,
        iv.center / iv.halfspan, 1e-8, 1e-5, _lib.ES_NONLIN_COMBUSTION, None, ptr(ws._scratch), ptr(ws_exp),
        ptr(ws_phi), nbytes, ctypes.byref(res), stream_handle())
for _ in range(20):
    lib.es_expeuler_step(*args)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    lib.es_expeuler_step(*args)
torch.cuda.synchronize()
print(f"C call alone per step {1e6 * (time.perf_counter() - t0) / n:.1f} us; kernel {res.series_ms * 1e3:.1f} us")
