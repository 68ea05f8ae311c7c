#!/usr/bin/env python
"""Benchmark of the fused Leja-stencil integrator step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3|C2|C1|C4|C5] [--impl b200|reference]

Default workload (N=1): BASELINE.json config 3 -- 512^3 7-point stencil,
homogeneous Dirichlet, combustion reaction term, exponential Rosenbrock-Euler
with Leja interpolation, fp64.  One "step" = one integrator step (device
resident state, all series, nonlinearity, Jacobian and step combination).

metric: Gpts.matvec/s = grid points x Newton-Leja nodes (matvecs) / second,
whole job (rows x nodes for the CSR config C5, where a step is one
phi1(-hA) v Newton-Leja action on a fixed v).  Also reported: the fused node kernel's achieved HBM GB/s against
MEASURED_PEAKS.json (roofline), the end-to-end number through the public API
with host buffers (e2e), the reference CPU path on the box's cores
(cpu_baseline), SM clocks during the timed region.

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference package with its compiled Cython core, built by
oracle/build_ref.sh; the plain-C oracle port if that is missing) on a bounded
sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "Gpts·matvec/s and HBM GB/s (% of peak) for Leja-stencil step at 1/2/4/8 B200"
UNIT = "Gpts·matvec/s"

CONFIGS = {
    "C3": dict(workload="512^3 7-point, homogeneous Dirichlet, combustion, exponential Rosenbrock-Euler + Leja",
               dims=(512, 512, 512), bc="homogeneous", coeff=None, method="rosenbrock", h=2.5e-5, tol=1e-4,
               bytes_per_node=40),
    "C2": dict(workload="4096^2 5-point, homogeneous Neumann, D=1/sqrt(1+x^2+y^2) (sampled once, streamed by TMA), "
                        "exp(-hA) v Leja action",
               dims=(4096, 4096, 1), bc="neumann", coeff="radial", method="linear", h=6e-7, tol=1e-4,
               bytes_per_node=32,
               roofline_note="algorithmic bytes exclude D (SURVEY 8(d)); the node also streams D: 40 B/pt moved"),
    "C1": dict(workload="256^2 5-point, homogeneous Dirichlet, combustion, exponential Euler + Leja",
               dims=(256, 256, 1), bc="homogeneous", coeff=None, method="euler", h=1e-4, tol=1e-4,
               bytes_per_node=32),
    "C4": dict(workload="1024^3 7-point, homogeneous Dirichlet, combustion, exponential Rosenbrock-Euler + Leja",
               dims=(1024, 1024, 1024), bc="homogeneous", coeff=None, method="rosenbrock", h=6.3e-6, tol=1e-4,
               bytes_per_node=40),
    "C5": dict(workload="CSR n=2^22 synthetic symmetric (6 U(-1,0) couplings/row mirrored, diagonal 12; 5.45e7 nnz), "
                        "phi1(-hA) v Newton-Leja action",
               kind="csr", n=2**22, per_row=6, dims=(2**22, 1, 1), bc=None, coeff=None, method="phi1", h=1.0,
               tol=1e-8, bytes_per_node=None),
}


def is_csr(cfg) -> bool:
    return cfg.get("kind") == "csr"


_CSR_CACHE: dict = {}


def csr_matrix(cfg):
    """The C5 operator (seeded, built once per process)."""
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    key = (cfg["n"], cfg["per_row"])
    if key not in _CSR_CACHE:
        _CSR_CACHE.clear()
        _CSR_CACHE[key] = synthetic_symmetric(cfg["n"], cfg["per_row"], seed=1234)
    return _CSR_CACHE[key]


def csr_node_bytes(n_rows: int, nnz: int) -> int:
    """Algorithmic bytes of one CSR Leja node: 8 vals + 4 col per
    nonzero, 8 (n+1) row_ptr, 8 n x, 8 n w', 16 n p."""
    return 12 * nnz + 40 * n_rows + 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the slab (NCCL) path even on one rank (tests the multi-GPU code path)")
    return ap.parse_args()


class _StdoutToStderr:
    """NCCL may print its version banner on stdout at communicator set-up;
    keep stdout for the one JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def initial_state(n: int, seed: int = 1234) -> np.ndarray:
    """u0 = 1 + 0.1 U[0, 1) (bench.py:112-114 seeding)."""
    return 1.0 + 0.1 * np.random.default_rng(seed).random(n)


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sms, mx, reasons = [], None, set()
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        loaded = [s for s in sms if s > 0.5 * max(sms)] or sms
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


# ---------------------------------------------------------------------------
# reference CPU path (bounded sample)


_REF_CACHE: dict = {}


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REPO, "oracle", "_ref", "expstencil"))


def reference_node_sample(cfg: dict, nodes: int):
    """Time `nodes` Newton-Leja nodes of the reference's newton_apply (its
    StencilOperator + compiled core) on the config's grid: returns
    (seconds, points*nodes, kind, threads, description).  The reference has
    no Neumann / Rosenbrock / in-kernel D: the series runs on its
    StencilOperator with the same grid (Dirichlet for Neumann, the sampled D
    array for the radial coefficient, A instead of A - diag g'), the closest
    cost-equivalent of the same hot loop."""
    if is_csr(cfg):
        return reference_csr_sample(cfg, nodes)
    nx, ny, nz = cfg["dims"]
    n = nx * ny * nz
    key = (tuple(cfg["dims"]), cfg["coeff"], nodes)
    if key not in _REF_CACHE:
        _REF_CACHE.clear()
        _REF_CACHE[key] = {"x": np.random.default_rng(1234).standard_normal(n)}
    cache = _REF_CACHE[key]
    x = cache["x"]
    if reference_available():
        sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
        os.environ.setdefault("EXPSTENCIL_KERNELS", "compiled")
        import expstencil as ref
        from expstencil import _kernels

        if "op" not in cache:
            coeff = (lambda X, Y, Z: 1.0 / np.sqrt(1.0 + X * X + Y * Y)) if cfg["coeff"] else None
            cache["op"] = ref.StencilOperator(ref.Grid3D(nx, ny, nz), ref.BoundaryCondition.homogeneous(),
                                              coeff=coeff)
            cache["it"] = ref.make_interpolant(ref.gershgorin_interval(cache["op"]), "phi1", -cfg["h"], nodes,
                                               cfg["tol"])
        op, it = cache["op"], cache["it"]
        t0 = time.perf_counter()
        _, mv = ref.newton_apply(op, it, x, 0.0)
        dt = time.perf_counter() - t0
        kind = "reference"
        desc = (f"reference newton_apply (expstencil {_kernels.default_backend()} core, oracle/_ref) on "
                f"{nx}x{ny}x{nz}, fixed degree {mv} (tol=0), phi1, Dirichlet A")
        threads = 1  # _core.pyx holds the GIL: the stencil runs on one core
    else:
        from oracle import oracle as orc

        spec = orc.StencilSpec(nx, ny, nz, coeff_kind=orc.COEFF_RADIAL if cfg["coeff"] else 0)
        lo, hi = spec.gershgorin()
        it = orc.interpolant(lo, hi, "phi1", -cfg["h"], nodes)
        t0 = time.perf_counter()
        _, mv = orc.newton_stencil(spec, it, x, 0.0)
        dt = time.perf_counter() - t0
        kind, threads = "port", orc.num_threads()
        desc = f"plain-C oracle port (OpenMP) newton series on {nx}x{ny}x{nz}, fixed degree {mv}"
    return dt, n * mv, kind, threads, desc


def reference_csr_sample(cfg: dict, nodes: int):
    """`nodes` fixed-degree Newton-Leja nodes of the reference's newton_apply
    on its own CsrMatrix of the C5 matrix (compiled core, one core)."""
    a = csr_matrix(cfg)
    n = a.nrows
    cache = _REF_CACHE.setdefault(("csr", n, nodes), {})
    if "x" not in cache:
        cache["x"] = np.random.default_rng(1234).standard_normal(n)
    x = cache["x"]
    if reference_available():
        sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
        os.environ.setdefault("EXPSTENCIL_KERNELS", "compiled")
        import expstencil as ref
        from expstencil import _kernels

        if "op" not in cache:
            cache["op"] = ref.CsrMatrix(n, n, a.row_ptr, a.col_idx, a.vals)
            cache["it"] = ref.make_interpolant(ref.gershgorin_interval(cache["op"]), "phi1", -cfg["h"], nodes,
                                               cfg["tol"])
        t0 = time.perf_counter()
        _, mv = ref.newton_apply(cache["op"], cache["it"], x, 0.0)
        dt = time.perf_counter() - t0
        kind, threads = "reference", 1
        desc = (f"reference newton_apply (expstencil {_kernels.default_backend()} core, oracle/_ref) on its "
                f"CsrMatrix n={n}, nnz={a.nnz}, fixed degree {mv} (tol=0), phi1")
    else:
        from oracle import oracle as orc

        oc = orc.Csr(n, a.row_ptr, a.col_idx, a.vals)
        lo, hi = oc.gershgorin()
        it = orc.interpolant(lo, hi, "phi1", -cfg["h"], nodes)
        t0 = time.perf_counter()
        _, mv = orc.newton_csr(oc, it, x, 0.0)
        dt = time.perf_counter() - t0
        kind, threads = "port", 1
        desc = f"plain-C oracle port newton series on CSR n={n}, nnz={a.nnz}, fixed degree {mv}"
    return dt, n * mv, kind, threads, desc


def reference_nodes_for(cfg: dict) -> int:
    if is_csr(cfg):
        return 8  # ~0.65 s per node on one core at 5.5e7 nonzeros

    n = int(np.prod(cfg["dims"]))
    # ~2 s per node at 512^3 on one core: keep each sample at ~10-30 s of CPU
    return max(2, min(40, int(3e8 // max(n, 1))))


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    nodes = reference_nodes_for(cfg)
    for _ in range(args.warmup if int(np.prod(cfg["dims"])) < 2**24 else min(args.warmup, 1)):
        reference_node_sample(cfg, nodes)
    times, units = [], 0
    kind = threads = desc = None
    for _ in range(args.steps):
        dt, u, kind, threads, desc = reference_node_sample(cfg, nodes)
        times.append(dt)
        units += u
    total = sum(times)
    value = units / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "grid": list(cfg["dims"]), "sample": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host_cpu_count": os.cpu_count(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm


def make_problem(cfg, es, world, use_dist):
    """(problem, n_local): one rank's slab of the config (the whole grid at N=1).
    u0 = 1 + 0.1 U[0,1) from numpy default_rng(1234) over the global grid (the
    same state at every N), or a partition-independent integer hash of the
    global index for grids too large for a host array per rank."""
    import torch

    from paper_1309_4616_b200.distributed import DistributedStencil, global_hash_state

    nx, ny, nz = cfg["dims"]
    g = es.Grid3D(nx, ny, nz)
    bc = es.BoundaryCondition.neumann() if cfg["bc"] == "neumann" else es.BoundaryCondition.homogeneous()
    op = es.StencilOperator(g, bc, coeff=es.radial_coeff if cfg["coeff"] == "radial" else None)
    nl = None if cfg["method"] == "linear" else es.combustion_g
    n = g.n
    if use_dist:
        op = DistributedStencil(op)
        lo, hi = op.comm.z_lo, op.comm.z_hi
    else:
        lo, hi = 0, nz
    plane = nx * ny
    if cfg["method"] == "linear":  # fixed series input v ~ N(0, 1)
        v = np.random.default_rng(1234).standard_normal(n)
        u0 = torch.from_numpy(v[lo * plane: hi * plane].copy()).cuda()
    elif n <= 2**28:
        u0 = torch.from_numpy(initial_state(n)[lo * plane: hi * plane].copy()).cuda()
    else:
        u0 = global_hash_state(nx, ny, nz, lo, hi, "cuda")
    return es.SemilinearProblem(operator=op, nonlinearity=nl, u0=u0), u0


def make_csr_problem(cfg, es, use_dist):
    """(operator, v): the C5 matrix (this rank's row block under torch.distributed)
    and the fixed series input v ~ N(0, 1) from default_rng(1234) over all rows."""
    import torch

    from paper_1309_4616_b200.distributed import DistributedCsr

    a = csr_matrix(cfg)
    v = np.random.default_rng(1234).standard_normal(a.nrows)
    if use_dist:
        op = DistributedCsr(a)
        v = v[op.comm.r_lo: op.comm.r_hi]
    else:
        op = a
    return op, torch.from_numpy(np.ascontiguousarray(v)).cuda()


class CsrStepper:
    """One phi1(-hA) v Newton-Leja action through the public API
    (es.newton_apply on a CsrMatrix / DistributedCsr); the input is fixed,
    the output is the action."""

    chain = False

    def __init__(self, cfg, es, op, use_dist=False):
        self.cfg, self.es, self.op, self.dist = cfg, es, op, use_dist
        self.h = cfg["h"]
        self.it = es.make_interpolant(es.gershgorin_interval(op), "phi1", -self.h, 150, cfg["tol"])

    def __call__(self, v, t):
        from paper_1309_4616_b200.integrator import StepStats

        p, mv = self.es.newton_apply(self.op, self.it, v)
        return p, StepStats(matvecs=mv)

    def launches(self, stats) -> int:
        # init + (node + slice reduce) per matvec + finalize; + round-0 kernel (p2p);
        # the NCCL row-block driver adds a decide per node
        ex = getattr(self.op, "exchange", "none")
        if ex == "nccl":
            return 3 * stats.matvecs + 2
        m = stats.matvecs
        if getattr(self.op, "two_node_passes", lambda: False)():
            m = (m + 1) // 2  # (node + reduce) per two-node pass
        return 2 * m + (3 if ex == "p2p" else 2)


class Stepper:
    """One integrator step of the configured method through the public API."""

    chain = True

    def __init__(self, cfg, es, problem, use_dist=False):
        self.cfg, self.es, self.problem, self.dist = cfg, es, problem, use_dist
        self.chain = cfg["method"] != "linear"  # linear: exp(-hA) v on a fixed v
        self.h, self.tol = cfg["h"], cfg["tol"]
        if cfg["method"] == "rosenbrock":
            self.ros = es.RosenbrockStepper(problem, self.tol)
        else:
            from paper_1309_4616_b200.integrator import _StepWorkspace

            self.ws = _StepWorkspace(problem, self.h, self.tol, 150)

    def __call__(self, u, t):
        if self.cfg["method"] == "rosenbrock":
            return self.ros.step(u, t, self.h)
        return self.ws.step(u, t)

    def launches(self, stats) -> int:
        """Kernels this step launched (counted from the code path).
        A TMA series = publish maps + init + (node + slice reduce) per node + finalize."""
        m = stats.matvecs
        ex = getattr(self.problem.operator, "exchange", "none")
        two = getattr(self.problem.operator, "two_node_passes", lambda: False)()
        if self.dist and ex == "p2p":
            # + the round-0 halo kernel; no NCCL per node; (node + slice) per pass
            series = (2 * ((m + 1) // 2) if two else 2 * m) + 4
        elif self.dist and ex == "nccl":
            series = 3 * m + 3  # node + slice reduce + decide per node (NCCL kernels not counted)
        elif two:
            series = 2 * ((m + 1) // 2) + 3  # two nodes per pass: (node + reduce) per pass
        else:
            series = 2 * m + 3
        if self.cfg["method"] == "rosenbrock":
            if self.ros._fused:
                return series + 2 + 1  # aux init + fused prologue; final axpy
            return series + 2 + 3 + 1 + 1 + 1  # combustion, Jacobian, A u, F axpy, final axpy
        if self.cfg["method"] == "linear":
            return series
        # two series (2 m + 6), combustion 2, axpy 1
        return series + 3 + 2 + 1


def measured_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def e2e_numpy_api(cfg, step, u, t, n, steps):
    """The same metric through the module-level public API with numpy arrays
    in and out -- the reference's calling convention (integrator.py:177-189,
    matfunc.py:271): pageable host copies inside the call, a fresh stepper /
    interpolant per call as `exponential_*_step` builds them.  Host-timed
    (perf_counter) around whole calls; a lower bound on what a numpy caller
    sees next to the pinned-buffer e2e above."""
    import time

    import torch

    import paper_1309_4616_b200 as es

    x = u.cpu().numpy()
    mv = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        if isinstance(step, Stepper):
            pr = step.problem
            if cfg["method"] == "rosenbrock":
                y, st = es.exponential_rosenbrock_step(pr, x, cfg["h"], cfg["tol"], t=t)
            else:
                y, st = es.exponential_euler_step(pr, x, cfg["h"], cfg["tol"], t=t)
            x = y if step.chain else x
        else:  # linear / CSR series on a fixed v
            op = getattr(step, "op", None)
            y, m = es.newton_apply(op, step.it, x)
            st = type("S", (), {"matvecs": m})
        mv += st.matvecs
        t += cfg["h"]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return {"value": float(n) * mv / dt / 1e9, "unit": UNIT, "steps": steps, "ms_per_step": 1e3 * dt / steps,
            "note": "module-level API, numpy in and out (pageable copies, per-call set-up), host-timed"}


def profiled_traffic(cfg_name: str):
    path = os.path.join(REPO, "profiles", "node_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(cfg_name)
    except (OSError, ValueError):
        return None


def config_block(args, cfg, n, world, nnz=None, replicas=False, exchange="p2p"):
    c = {"workload": cfg["workload"], "config": args.config, "method": cfg["method"], "h": cfg["h"],
         "tol": cfg["tol"]}
    via = ("NVLink peer memory, fused into the node kernels" if exchange == "p2p"
           else "NCCL, host-driven per node")
    if nnz is not None:
        c.update({"rows": n, "nnz": nnz,
                  "parallelism": f"row blocks x{world} (all-gather of w over {via})" if world > 1 else "single",
                  "l2": f"matrix ({12 * nnz / 2**20:.0f} MiB of vals+col) streams from HBM, larger than L2; "
                        f"the {8 * n / 2**20:.0f} MiB vectors are L2-resident by design (no flush)"})
        return c
    c.update({"grid": list(cfg["dims"]), "bc": cfg["bc"], "coeff": cfg["coeff"],
              "parallelism": ("single" if world == 1 else
                              f"replicas x{world} (a single-plane grid cannot be slab-partitioned, "
                              f"decomp.py:76-77)" if replicas else
                              f"z-slabs x{world} (halo planes and norm slices over {via})"),
              "l2": f"inputs larger than L2 ({8 * n / 2**20:.0f} MiB per vector)" if 8 * n >= 2**27
              else "working set inside L2 (no flush)"})
    return c


def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1309_4616_b200 as es
    from paper_1309_4616_b200 import timing

    rank, world, local = dist_env()
    if torch.cuda.device_count() <= local:
        raise RuntimeError(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} CUDA device(s)")
    torch.cuda.set_device(local)
    use_dist = world > 1 or args.force_dist
    # single-plane grids (C1, C2) cannot be slab-partitioned (decomp.py:76-77):
    # every rank runs the whole problem as an independent replica
    replicas = world > 1 and not is_csr(cfg) and cfg["dims"][2] == 1
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        with _StdoutToStderr():
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
            dist.barrier()
    nx, ny, nz = cfg["dims"]
    n = nx * ny * nz  # global points (rows for CSR)
    if is_csr(cfg):
        op, u0 = make_csr_problem(cfg, es, use_dist)
        step = CsrStepper(cfg, es, op, use_dist)
        nnz_local = int(op.vals.shape[0]) if use_dist else op.nnz
        bytes_node = csr_node_bytes(u0.numel(), nnz_local)
        nnz_total = csr_matrix(cfg).nnz
    else:
        problem, u0 = make_problem(cfg, es, world, use_dist and not replicas)
        step = Stepper(cfg, es, problem, use_dist and not replicas)
        bytes_node = cfg["bytes_per_node"] * u0.numel()
    n_local = u0.numel()

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    dist_op = step.op if is_csr(cfg) else step.problem.operator
    ledger = getattr(dist_op, "ledger", None) if use_dist and not replicas else None

    u = u0.clone()
    t = 0.0
    for _ in range(args.warmup):
        out, _ = step(u, t)
        u = out if step.chain else u
        t += cfg["h"]
    barrier()
    # ---- device-resident timed region ----
    matvecs, launches = 0, 0
    moved0 = ledger.bytes_total if ledger is not None else 0
    with ClockSampler(local) as clocks, timing.SeriesTimer() as tm:
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            out, st = step(u, t)
            u = out if step.chain else u
            t += cfg["h"]
            matvecs += st.matvecs
            launches += step.launches(st)
        ev1.record()
        barrier()
    elapsed = ev0.elapsed_time(ev1) * 1e-3
    series_s, series_mv = tm.totals()
    t_max = elapsed
    units = float(n_local) * matvecs
    if world > 1:
        buf = torch.tensor([elapsed, units], dtype=torch.float64, device="cuda")
        tmax = buf[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        usum = buf[1:].clone()
        dist.all_reduce(usum, op=dist.ReduceOp.SUM)
        t_max, units = float(tmax.item()), float(usum.item())
    value = units / t_max / 1e9
    # inter-GPU traffic of the timed region: the reference's ledger formula
    # (2 (m-1) nx ny halo / (m-1) n all-gather scalars per node), whole job
    nvlink = None
    if ledger is not None and world > 1:
        moved = float(ledger.bytes_total - moved0)
        peer_gbs = 900.0  # NVLink 5 per GPU per direction
        nvlink = {"bytes_per_step": moved / args.steps, "GB/s": moved / t_max / 1e9,
                  "per_gpu_GB/s": moved / t_max / 1e9 / world,
                  "frac_of_900GBs_per_gpu": moved / t_max / 1e9 / world / peer_gbs,
                  "note": "ledger bytes (halo planes / gathered vector slices) over the device-timed region"}

    # roofline of the dominant kernel: the fused node (series time / nodes),
    # or the two-node pass (series time / passes) where the series uses it
    node_s = series_s / max(series_mv, 1)
    peak, peak_src = measured_peak()
    two = not is_csr(cfg) and getattr(step.problem.operator, "two_node_passes", lambda: False)()
    if two:
        passes = max(tm.passes(), 1)
        two_p, one_p = tm.pass_mix()
        launch_s = series_s / passes
        # a two-node pass reads w, p (+g') and writes w'', p'' -- and p' only
        # where the series could stop at its first node (tol > 0 with the
        # one-node tail pass disabled, ES_TB_TAIL=0; csrc/series.cuh
        # tb_store_pk); the one-node tail pass reads w, p (+g') and writes w', p'
        pk_stored = cfg["tol"] > 0 and os.environ.get("ES_TB_TAIL", "1") == "0"
        bytes_all = (two_p * (cfg["bytes_per_node"] + (8 if pk_stored else 0)) + one_p * cfg["bytes_per_node"]) * n_local
        bytes_launch = bytes_all / passes
        achieved = bytes_launch / launch_s / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": profiled_traffic(args.config + "_tb"),
                    "kernel": ("k_node_tb2m (two fused Leja nodes per HBM pass, row-marching 2D)" if cfg["dims"][2] == 1
                               else "k_node_tb3m (two fused Leja nodes per HBM pass, plane-marching 3D)"),
                    "bytes_per_launch": bytes_launch,
                    "bytes_per_point": bytes_launch / n_local, "launch_us": launch_s * 1e6, "launches": passes,
                    "two_node_passes": two_p, "one_node_passes": one_p,
                    "node_us": node_s * 1e6,
                    "one_node_equiv_GBs": bytes_node / node_s / 1e9,
                    "note": "one-node algorithmic bytes (SURVEY 8(d)) per node time; above the HBM peak because "
                            "two nodes share one pass",
                    "peak_source": peak_src, "series_share_of_step": series_s / elapsed if elapsed > 0 else None}
    else:
        achieved = bytes_node / node_s / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": profiled_traffic(args.config),
                    "kernel": "k_csr_node (fused CSR Leja node)" if is_csr(cfg) else "k_node_tma (fused Leja node)",
                    "bytes_per_node": bytes_node,
                    "bytes_per_point": bytes_node / n_local, "node_us": node_s * 1e6, "peak_source": peak_src,
                    "series_share_of_step": series_s / elapsed if elapsed > 0 else None}
        if cfg.get("roofline_note"):
            roofline["note"] = cfg["roofline_note"]

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        pin_in = torch.from_numpy(u.cpu().numpy()).pin_memory()
        pin_out = torch.empty_like(pin_in).pin_memory()
        fixed_in = pin_in
        e2e_steps = max(3, args.steps // 2)
        mv_e2e = 0
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(e2e_steps):
            ud = pin_in.to("cuda", non_blocking=True)
            ud, st = step(ud, t)
            t += cfg["h"]
            pin_out.copy_(ud, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            pin_in, pin_out = (pin_out, pin_in) if step.chain else (fixed_in, pin_out)
            mv_e2e += st.matvecs
        e1.record()
        barrier()
        e_el = e0.elapsed_time(e1) * 1e-3
        e_units = float(n) * mv_e2e * (world if replicas else 1)
        if world > 1:
            b = torch.tensor([e_el], dtype=torch.float64, device="cuda")
            dist.all_reduce(b, op=dist.ReduceOp.MAX)
            e_el = float(b.item())
        nb = 8 * n * (world if replicas else 1)
        e2e = {"value": e_units / e_el / 1e9, "unit": UNIT, "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "steps": e2e_steps, "ms_per_step": 1e3 * e_el / e2e_steps}
        if is_csr(cfg):
            e2e["note"] = "the matrix is uploaded once (operator set-up); each step copies v in and p out"
        if world > 1:
            e2e["note"] = "each rank copies its own slab; bytes are whole-job"
        if world == 1:
            e2e["api_numpy"] = e2e_numpy_api(cfg, step, u, t, n, e2e_steps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nodes = reference_nodes_for(cfg)
        dt, u_cpu, kind, threads, desc = reference_node_sample(cfg, nodes)
        cpu = {"value": u_cpu / dt / 1e9, "unit": UNIT, "cores": threads, "kind": kind, "sample": desc,
               "seconds": dt, "host_cpu_count": os.cpu_count()}

    gpus_active = 1
    if world > 1:  # distinct physical devices the ranks ran on
        uuids = [None] * world
        dist.all_gather_object(uuids, str(torch.cuda.get_device_properties(local).uuid))
        gpus_active = len(set(uuids))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "gpus_active": gpus_active,
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 and not replicas else "weak", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic: seeded symmetric CSR (default_rng(1234)), v ~ N(0,1) default_rng(1234)"
                     if is_csr(cfg) else
                     "synthetic: fixed v ~ N(0,1), numpy default_rng(1234)" if cfg["method"] == "linear" else
                     "synthetic: u0 = 1 + 0.1 U[0,1), numpy default_rng(1234) over the global grid" if n <= 2**28
                     else "synthetic: u0 = 1 + 0.1 hash(global index)"),
            "config": config_block(args, cfg, n, world, nnz_total if is_csr(cfg) else None, replicas,
                                   getattr(step.op if is_csr(cfg) else step.problem.operator, "exchange", "p2p")),
            "matvecs_per_step": matvecs / args.steps, "steps_per_s": args.steps / t_max,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
            "gpu_launches": launches,
            "nvlink": nvlink,
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


def self_launch(args) -> int:
    """`bench.py --gpus N` run without a launcher: start N ranks (one process
    per GPU) under torch.distributed.run on 127.0.0.1 and pass their exit
    code through; rank 0 prints the JSON line."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible",
              file=sys.stderr, flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = dist_env()[1]
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop the launcher", file=sys.stderr, flush=True)
        sys.exit(2)
    run_b200(args, cfg)


if __name__ == "__main__":
    main()
