"""Probe the GPU box: host RAM, cores, pinned H2D / D2H / D2D bandwidth."""
import os, subprocess, json, time
import torch
out = {}
out["cpu_count"] = os.cpu_count()
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500]
    out["free"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
    out["smi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
except Exception as e:
    out["err"] = str(e)
dev = torch.device("cuda:0")
def bw(nbytes, kind):
    if kind == "h2d":
        src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True); dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    elif kind == "d2h":
        src = torch.empty(nbytes, dtype=torch.uint8, device=dev); dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    else:
        src = torch.empty(nbytes, dtype=torch.uint8, device=dev); dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    best = 0
    for _ in range(6):
        with torch.cuda.stream(s):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); dst.copy_(src, non_blocking=True); b.record(s)
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best
for mb in (9.44, 64, 1024):
    n = int(mb * 1e6)
    out[f"h2d_{mb}MB_GBs"] = bw(n, "h2d")
    out[f"d2h_{mb}MB_GBs"] = bw(n, "d2h")
# pinned alloc speed for 8 GB
t = time.time(); big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True); out["pin8GB_s"] = time.time() - t
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
