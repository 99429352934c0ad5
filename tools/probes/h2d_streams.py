"""H2D throughput of 128 expert-sized (9.44 MB) pinned->device copies: one copy
stream vs two alternating streams, with/without an event after each copy."""
import torch

n, sz = 128, 3 * 768 * 2048 * 2
h = torch.empty(n * sz, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n * sz, dtype=torch.uint8, device="cuda")
s = [torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()]


def run(nstreams, events):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for st in s[:nstreams]:
        st.wait_stream(torch.cuda.current_stream())
    for i in range(n):
        st = s[i % nstreams]
        with torch.cuda.stream(st):
            d[i * sz:(i + 1) * sz].copy_(h[i * sz:(i + 1) * sz], non_blocking=True)
            if events:
                torch.cuda.Event().record(st)
    for st in s[:nstreams]:
        torch.cuda.current_stream().wait_stream(st)
    b.record()
    b.synchronize()
    return n * sz / (a.elapsed_time(b) * 1e-3) / 1e9


for it in range(2):
    for ns in (1, 2, 3):
        for ev in (False, True):
            print(f"streams={ns} events={ev}: {run(ns, ev):.1f} GB/s")
big = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
big[0].record()
d.copy_(h, non_blocking=True)
big[1].record()
big[1].synchronize()
print(f"one 1.2 GB copy: {n * sz / (big[0].elapsed_time(big[1]) * 1e-3) / 1e9:.1f} GB/s")

# with a stream memory op (ready-flag write) after each copy, as the copy runtime does
from cuda.bindings import driver as cu

flags = torch.zeros(n, dtype=torch.int32, device="cuda")


def run_wv(nostall):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = s[0]
    a.record()
    st.wait_stream(torch.cuda.current_stream())
    fl = cu.CUstreamWriteValue_flags.CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER if nostall else \
        cu.CUstreamWriteValue_flags.CU_STREAM_WRITE_VALUE_DEFAULT
    for i in range(n):
        with torch.cuda.stream(st):
            d[i * sz:(i + 1) * sz].copy_(h[i * sz:(i + 1) * sz], non_blocking=True)
        cu.cuStreamWriteValue32(st.cuda_stream, flags.data_ptr() + 4 * i, i + 1, fl)
    torch.cuda.current_stream().wait_stream(st)
    b.record()
    b.synchronize()
    return n * sz / (a.elapsed_time(b) * 1e-3) / 1e9


for it in range(2):
    print(f"1 stream + writeValue32 (barrier): {run_wv(False):.1f} GB/s; no barrier: {run_wv(True):.1f} GB/s")


def run_wv2(ns):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for st in s[:ns]:
        st.wait_stream(torch.cuda.current_stream())
    for i in range(n):
        st = s[i % ns]
        with torch.cuda.stream(st):
            d[i * sz:(i + 1) * sz].copy_(h[i * sz:(i + 1) * sz], non_blocking=True)
        cu.cuStreamWriteValue32(st.cuda_stream, flags.data_ptr() + 4 * i, i + 1,
                                cu.CUstreamWriteValue_flags.CU_STREAM_WRITE_VALUE_DEFAULT)
    for st in s[:ns]:
        torch.cuda.current_stream().wait_stream(st)
    b.record()
    b.synchronize()
    return n * sz / (a.elapsed_time(b) * 1e-3) / 1e9


for it in range(2):
    print(f"2 streams + writeValue32 (barrier): {run_wv2(2):.1f} GB/s; 3 streams: {run_wv2(3):.1f} GB/s")
