#!/bin/bash
# Round-2 micro measurements (run under gpurun): prune / glue / skinny timings and
# ncu captures of the kernels the verdict named (prune R=1 and R=256, router R=1).
O=gpurun_out/r02micro
mkdir -p $O
timeout 300 python tools/bench_prune.py 1 8 64 256 > $O/prune.log 2>&1
timeout 300 python tools/bench_small.py 1 > $O/small_R1.log 2>&1
timeout 300 python tools/bench_small.py 256 > $O/small_R256.log 2>&1
timeout 300 python tools/bench_skinny.py 8 > $O/skinny8.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prune -s 5 -c 1 \
  -o $O/ncu_prune_R1 python tools/bench_prune.py 1 > $O/ncu_prune_R1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prune -s 5 -c 1 \
  -o $O/ncu_prune_R256 python tools/bench_prune.py 256 > $O/ncu_prune_R256.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route -s 2 -c 2 \
  -o $O/ncu_route_R1 python tools/bench_small.py 1 > $O/ncu_route_R1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:skinny -s 2 -c 1 \
  -o $O/ncu_skinny python tools/bench_skinny.py 8 > $O/ncu_skinny.log 2>&1
ls -la $O
