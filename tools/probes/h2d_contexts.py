"""Is the ~55 GB/s pinned H2D ceiling per CUDA context or per link?

One process, driver API (cuda-python): the primary context A and a second
context B on the same device (cuCtxCreate).  One portable pinned host buffer
(cuMemHostAlloc PORTABLE: page-locked for every context), a device buffer per
context, one stream per context.  Measures (wall clock around both streams'
completion, best of 3):
  A alone, B alone, A and B at once (each copies half), and 1/2/4 streams in A.
Then two PROCESSES with a synchronised start (a file barrier) copying for the
same window.

    python tools/probes/h2d_contexts.py
"""
import json
import os
import subprocess
import sys
import time

from cuda.bindings import driver as cu

GiB = 1 << 30


def ok(r):
    if isinstance(r, tuple):
        assert r[0] == cu.CUresult.CUDA_SUCCESS, r
        return r[1] if len(r) == 2 else r[1:]
    assert r == cu.CUresult.CUDA_SUCCESS, r
    return None


def single_process():
    ok(cu.cuInit(0))
    dev = ok(cu.cuDeviceGet(0))
    ctx_a = ok(cu.cuDevicePrimaryCtxRetain(dev))
    ok(cu.cuCtxSetCurrent(ctx_a))
    n = 2 * GiB
    h = ok(cu.cuMemHostAlloc(n, cu.CU_MEMHOSTALLOC_PORTABLE))
    d_a = ok(cu.cuMemAlloc(n))
    streams_a = [ok(cu.cuStreamCreate(cu.CUstream_flags.CU_STREAM_NON_BLOCKING)) for _ in range(4)]
    ctx_b = ok(cu.cuCtxCreate(0, dev))
    ok(cu.cuCtxSetCurrent(ctx_b))
    d_b = ok(cu.cuMemAlloc(n))
    s_b = ok(cu.cuStreamCreate(cu.CUstream_flags.CU_STREAM_NON_BLOCKING))
    ok(cu.cuCtxSetCurrent(ctx_a))

    def run(jobs, reps=3):
        """jobs: list of (ctx, stream, dst, src_off, nbytes); wall time until all done."""
        best = 0.0
        total = sum(j[4] for j in jobs)
        for _ in range(reps):
            for c, _, _, _, _ in jobs:
                ok(cu.cuCtxSetCurrent(c))
                ok(cu.cuCtxSynchronize())
            t0 = time.perf_counter()
            for c, st, dst, off, nb in jobs:
                ok(cu.cuCtxSetCurrent(c))
                ok(cu.cuMemcpyHtoDAsync(int(dst) + off, int(h) + off, nb, st))
            for c, st, _, _, _ in jobs:
                ok(cu.cuCtxSetCurrent(c))
                ok(cu.cuStreamSynchronize(st))
            best = max(best, total / (time.perf_counter() - t0) / 1e9)
        ok(cu.cuCtxSetCurrent(ctx_a))
        return best

    out = {}
    out["A_alone_2GiB"] = run([(ctx_a, streams_a[0], d_a, 0, n)])
    out["B_alone_2GiB"] = run([(ctx_b, s_b, d_b, 0, n)])
    out["A_and_B_1GiB_each"] = run([(ctx_a, streams_a[0], d_a, 0, GiB), (ctx_b, s_b, d_b, GiB, GiB)])
    for k in (2, 4):
        part = n // k
        out[f"A_{k}_streams"] = run([(ctx_a, streams_a[i], d_a, i * part, part) for i in range(k)])
    return out


def proc_child(path, secs):
    import torch

    n = GiB
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d.copy_(h)
    torch.cuda.synchronize()
    open(path + f".{os.getpid()}", "w").close()
    while len([f for f in os.listdir(os.path.dirname(path)) if f.startswith(os.path.basename(path) + ".")]) < 2:
        time.sleep(0.001)
    t0, k = time.perf_counter(), 0
    while time.perf_counter() - t0 < secs:
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        k += 1
    print(json.dumps({"gbs": k * n / (time.perf_counter() - t0) / 1e9}))


def two_processes(secs=4.0):
    import tempfile

    tmp = tempfile.mkdtemp()
    path = os.path.join(tmp, "bar")
    ps = [subprocess.Popen([sys.executable, __file__, "child", path, str(secs)], stdout=subprocess.PIPE, text=True)
          for _ in range(2)]
    res = [json.loads(p.communicate()[0].strip().splitlines()[-1])["gbs"] for p in ps]
    return {"two_processes_each": res, "two_processes_sum": sum(res)}


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        proc_child(sys.argv[2], float(sys.argv[3]))
        sys.exit(0)
    out = single_process()
    out.update(two_processes())
    print(json.dumps(out, indent=1))
