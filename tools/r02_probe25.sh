#!/bin/bash
# prefix glue without torch elementwise kernels: parity tests + launch list of one step
O=gpurun_out/probe25; mkdir -p $O
timeout 1500 python -m pytest -q -x tests/test_gpu_headline.py tests/test_gpu_stack.py tests/test_gpu_ep.py tests/test_gpu_compress.py tests/test_gpu_compress_props.py tests/test_gpu_predict.py > $O/tests.txt 2>&1; tail -3 $O/tests.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python tools/timeline_step.py 64 c3_qwen3vl 1 > $O/tl.log 2>&1
python - <<'PY'
import csv, re
rows = list(csv.reader(open("gpurun_out/probe25/launches.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki = h.index("Kernel Name"); ii = h.index("ID")
seen, names = set(), []
for r in rows[hi + 1:]:
    if len(r) < len(h): continue
    if r[ii] in seen: continue
    seen.add(r[ii]); names.append(re.sub(r"^void ", "", r[ki])[:70])
pi = [j for j, n in enumerate(names) if n.startswith("<unnamed>::prune_kernel") or n.startswith("prune_kernel")]
j = pi[-1]
print("kernels around the prune of the last forward:")
for n in names[j - 12:j + 22]: print("  ", n)
PY
