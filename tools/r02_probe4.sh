#!/bin/bash
# phase profiles (prof build) of prune / split router, skinny decode FFN timing, H2D link probe
O=gpurun_out/probe4
mkdir -p $O
export VMM_LIB=$PWD/paper_2605_05899_b200/libvismmoe_prof.so
for R in 1 8 256; do echo "== prune R=$R"; timeout 120 python tools/prune_prof.py $R; done > $O/prune_prof.txt 2>&1
for n in 1216 2368; do for la in 0 1; do echo "== route N=$n la=$la"; timeout 120 python tools/route_prof.py $n $la; done; done > $O/route_prof.txt 2>&1
unset VMM_LIB
timeout 300 python tools/bench_prune.py 1 8 64 256 > $O/prune_times.txt 2>&1
timeout 300 python tools/bench_skinny.py 8 > $O/skinny8.txt 2>&1
timeout 600 python tools/probes/h2d_probe.py > $O/h2d_probe.json 2>&1
cat $O/prune_prof.txt $O/route_prof.txt $O/prune_times.txt $O/skinny8.txt $O/h2d_probe.json | head -150
