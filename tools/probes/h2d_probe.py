"""Host->device link probe: what limits the pinned-pool expert copies?

An early two-process run suggested 43 GB/s EACH (87 GB/s total); that was an
artefact of unsynchronised timing windows -- with a synchronised start two
processes get 27.7 GB/s each, 55.4 GB/s together, and a second CUDA context
in one process adds nothing either (tools/probes/h2d_contexts.py,
profiles/r02_h2d_contexts.json): ~55.5 GB/s is the link.  This probe measures,
in one process:
  A  one 1 GiB copy                                        (copy engine, 1 stream)
  B  1 GiB split over N streams, N = 2/4/8                (several copy engines)
  C  N streams from N SEPARATELY pinned buffers            (host memory placement)
  D  expert-sized (9.44 MB) copies round-robin on N streams
  E  an SM kernel reading the mapped pinned pool (zero-copy) with all SMs
plus the GPU's PCIe link from nvidia-smi and the host NUMA layout.
"""
import json
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

GiB = 1 << 30
SZ = 3 * 768 * 2048 * 2


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed(fn, reps=3):
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        nbytes = fn()
        b.record()
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


_KSRC = r"""
extern "C" __global__ void zc_copy(const int4 *__restrict__ src, int4 *__restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
"""


def zero_copy(h, d, blocks_per_sm):
    from cuda.bindings import driver as cu, nvrtc

    prog = nvrtc.nvrtcCreateProgram(_KSRC.encode(), b"zc.cu", 0, [], [])[1]
    opts = [b"--gpu-architecture=sm_100a"]
    assert nvrtc.nvrtcCompileProgram(prog, len(opts), opts)[0] == nvrtc.nvrtcResult.NVRTC_SUCCESS
    n = nvrtc.nvrtcGetCUBINSize(prog)[1]
    buf = b" " * n
    nvrtc.nvrtcGetCUBIN(prog, buf)
    mod = cu.cuModuleLoadData(buf)[1]
    fn = cu.cuModuleGetFunction(mod, b"zc_copy")[1]
    import ctypes
    import numpy as np

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nvec = GiB // 16
    a_src = np.array([h.data_ptr()], dtype=np.uint64)
    a_dst = np.array([d.data_ptr()], dtype=np.uint64)
    a_n = np.array([nvec], dtype=np.int64)
    args = np.array([a.ctypes.data for a in (a_src, a_dst, a_n)], dtype=np.uint64)

    def run():
        st = torch.cuda.current_stream().cuda_stream
        r = cu.cuLaunchKernel(fn, sms * blocks_per_sm, 1, 1, 512, 1, 1, 0, st, args.ctypes.data, 0)
        assert r[0] == cu.CUresult.CUDA_SUCCESS, r
        return GiB

    v = timed(run)
    torch.cuda.synchronize()
    assert bool((d[:GiB] == h[:GiB].to("cuda")).all())
    return v


def main():
    out = {}
    try:
        out["nvidia_smi_pcie"] = subprocess.run(
            ["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,"
             "pcie.link.width.max", "--format=csv"], capture_output=True, text=True).stdout.strip()
        out["numa"] = subprocess.run(["bash", "-c", "lscpu | grep -i -E 'numa|socket|model name'"],
                                     capture_output=True, text=True).stdout.strip()
        out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout.strip()[:2000]
    except Exception as e:  # noqa: BLE001
        out["smi_error"] = str(e)
    h = torch.empty(2 * GiB, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(2 * GiB, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(8)]
    cur = torch.cuda.current_stream()

    def split_copy(n, srcs=None, total=GiB):
        for st in streams[:n]:
            st.wait_stream(cur)
        part = total // n
        for i in range(n):
            src = srcs[i] if srcs else h[i * part:(i + 1) * part]
            with torch.cuda.stream(streams[i]):
                d[i * part:(i + 1) * part].copy_(src[:part], non_blocking=True)
        for st in streams[:n]:
            cur.wait_stream(st)
        return total

    out["A_one_1GiB_copy"] = timed(lambda: split_copy(1))
    for n in (2, 4, 8):
        out[f"B_1GiB_over_{n}_streams"] = timed(lambda n=n: split_copy(n))
    sep = [torch.empty(GiB // 4, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
    for n in (2, 4):
        out[f"C_{n}_separate_pinned_buffers"] = timed(lambda n=n: split_copy(n, sep, total=n * (GiB // 4)))
    nexp = (2 * GiB) // SZ

    def experts(n):
        for st in streams[:n]:
            st.wait_stream(cur)
        for i in range(nexp):
            with torch.cuda.stream(streams[i % n]):
                d[i * SZ:(i + 1) * SZ].copy_(h[i * SZ:(i + 1) * SZ], non_blocking=True)
        for st in streams[:n]:
            cur.wait_stream(st)
        return nexp * SZ

    for n in (1, 2, 4, 8):
        out[f"D_expert_copies_{n}_streams"] = timed(lambda n=n: experts(n))
    # E: SM-driven zero-copy read of the pinned buffer (UVA: the pinned host pointer is
    # device-accessible): a grid-stride int4 copy kernel compiled with NVRTC, all SMs
    try:
        for blocks_per_sm in (2, 4, 8):
            out[f"E_zero_copy_kernel_{blocks_per_sm}_ctas_per_sm"] = zero_copy(h, d, blocks_per_sm)
    except Exception as e:  # noqa: BLE001
        out["E_zero_copy"] = f"skipped: {e}"
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
