import os, sys
sys.path.insert(0, "/root/repo")
import torch, paper_1309_4616_b200 as es
from paper_1309_4616_b200.sparse import synthetic_symmetric
m = synthetic_symmetric(65536, 3, seed=1)
it = es.make_interpolant(es.gershgorin_interval(m), "phi1", -1.0, 40, 1e-8)
v = torch.randn(m.nrows, dtype=torch.float64, device="cuda")
for _ in range(3): es.newton_apply(m, it, v, 0.0)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); p, mv = es.newton_apply(m, it, v, 0.0); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) * 1e3 / mv)
print(f"csr 65536 node {best:.1f} us", flush=True)
