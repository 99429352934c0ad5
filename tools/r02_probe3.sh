#!/bin/bash
# FFN timing A/B, alternating configs (lag, hints) three rounds
O=gpurun_out/probe3
mkdir -p $O
for rep in 1 2 3; do
for cfg in "4 0" "4 3" "2 1" "2 3" "3 3"; do
  set -- $cfg
  t=$(VMM_FFN_LAG=$1 VMM_FFN_L2HINTS=$2 FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 256 2>&1 | tail -1)
  echo "rep=$rep lag=$1 hints=$2 $t" >> $O/summary.txt
done; done
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv >> $O/summary.txt
cat $O/summary.txt
