"""Build libvismmoe.so (sm_100a) in-tree with nvcc/g++.

    python -m paper_2605_05899_b200.build        # or __graft_entry__.build()

Objects go to paper_2605_05899_b200/_build/, the library next to this file so
it travels with the repo snapshot to the GPU box.  Decision kernels (prune,
predictors) are compiled with -fmad=false and the host policy with
-ffp-contract=off so every fp64 op rounds exactly like the CPython reference.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# VMM_BUILD_VARIANT=prof: dev build with the FFN wait counters (-DVMM_FFN_PROF) into
# _build_prof/ and libvismmoe_prof.so (load it with VMM_LIB=...; tools/ffn_prof.py)
VARIANT = os.environ.get("VMM_BUILD_VARIANT", "")
OUT = os.path.join(HERE, "_build" + (f"_{VARIANT}" if VARIANT else ""))
LIB = os.path.join(HERE, "libvismmoe" + (f"_{VARIANT}" if VARIANT else "") + ".so")
DEFS = {"prof": ["-DVMM_FFN_PROF", "-DVMM_PRUNE_PROF"]}.get(VARIANT, [])
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU = {
    "prune.cu": ["-fmad=false"],
    "predict.cu": ["-fmad=false"],
    "route.cu": [],
    "route_sm100.cu": [],
    "sm100.cu": [],
    "permute.cu": [],
    "ffn_sm100.cu": [],
    "diag.cu": ["-fmad=false"],
    "ep.cu": [],
}
CPP = ["engine.cpp", "xfer.cpp", "capi.cpp", "stack.cpp"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def _stale(obj, src):
    deps = [src, os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "sm100.cuh"),
            os.path.join(HERE, "..", "include", "vismmoe.h")]
    return not os.path.exists(obj) or any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    nvcc = _nvcc()
    inc = ["-I", os.path.join(HERE, "..", "include")]
    jobs = []
    for src, extra in CU.items():
        obj = os.path.join(OUT, src + ".o")
        cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
               *extra, *DEFS, *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        jobs.append((obj, os.path.join(CSRC, src), cmd))
    for src in CPP:
        obj = os.path.join(OUT, src + ".o")
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-I/usr/local/cuda/include", *inc,
               "-c", os.path.join(CSRC, src), "-o", obj]
        jobs.append((obj, os.path.join(CSRC, src), cmd))
    todo = [j for j in jobs if force or _stale(j[0], j[1])]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for (obj, _, cmd), log in zip(todo, ex.map(lambda j: _run(j[2]), todo)):
            if verbose and log:
                print(log, file=sys.stderr)
    objs = [j[0] for j in jobs]
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        _run([nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-ldl", "-lpthread", "-lrt"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
