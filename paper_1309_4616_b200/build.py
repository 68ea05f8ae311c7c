"""Build libexpstencil_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1309_4616_b200.build      (or __graft_entry__.build())

The library is plain C ABI (include/expstencil_b200.h) over a static CUDA
runtime, so it loads into any process (ctypes) and shares the primary
context -- and therefore device pointers and streams -- with PyTorch.
-fmad=false keeps every fp64 expression uncontracted (bitwise parity with the
reference's -ffp-contract=off core); -lineinfo maps ncu source pages.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libexpstencil_b200.so")
SOURCES = ["capi.cu", "stencil.cu", "csr.cu", "pointwise.cu", "graph.cu", "f32.cu", "step.cu", "csr_generic.cu", "series_small.cu"]
HEADERS = ["es_common.cuh", "es_host.h", "stencil.cuh", "series.cuh", "stencil_tma.cuh", "stencil_tb.cuh",
           "stencil_tb2d.cuh", "stencil_tb2m.cuh", "stencil_tb3m.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-fmad=false", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xptxas", "-O3",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build expstencil_b200")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    # every file under csrc/ (a header missing from HEADERS must not leave a stale build)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(REPO, "include", "expstencil_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    cc = nvcc()
    cmds, objs = [], []
    for src in SOURCES:
        obj = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
        cmd = [cc, *ARCH, *NVCC_FLAGS, *os.environ.get("ES_NVCC_EXTRA", "").split(), "-I", os.path.join(REPO, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        cmds.append(cmd)
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(len(cmds)) as pool:
        for r in pool.map(lambda c: subprocess.run(c, check=False), cmds):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    tmp = LIB + ".tmp"
    subprocess.run([cc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lrt", "-ldl", "-lpthread"],
                   check=True)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
