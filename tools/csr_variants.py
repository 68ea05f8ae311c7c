"""Time the CSR Leja node variants (ES_CSR_VARIANT) on the C5 matrix:
fixed-degree series (tol = 0), CUDA events around each series, node time =
series time / nodes.  Checks every variant's p bitwise against variant 0.
Not part of the product."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1309_4616_b200 as es  # noqa: E402
from paper_1309_4616_b200.sparse import synthetic_symmetric  # noqa: E402

variants = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,6,5,9,12").split(",")]
m = synthetic_symmetric(2**22, 6, seed=1234)
nodes = 30
it = es.make_interpolant(es.gershgorin_interval(m), "phi1", -1.0, nodes, 1e-8)
v = torch.randn(m.nrows, dtype=torch.float64, device="cuda")
bytes_node = 12 * m.nnz + 40 * m.nrows + 8
ref = None
for var in variants:
    os.environ["ES_CSR_VARIANT"] = str(var)
    for _ in range(2):
        p, mv = es.newton_apply(m, it, v, 0.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p, mv = es.newton_apply(m, it, v, 0.0)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / mv)
    t = min(ts)
    same = ref is None or torch.equal(p, ref)
    ref = p if ref is None else ref
    print(f"variant {var}: node {t * 1e6:.1f} us  {bytes_node / t / 1e9:.0f} GB/s algorithmic  bitwise={same}",
          flush=True)
