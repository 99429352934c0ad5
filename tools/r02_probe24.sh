#!/bin/bash
O=gpurun_out/probe24; mkdir -p $O
for rep in 1 2 3; do for lag in 4 5 6; do
  echo "rep=$rep lag=$lag $(VMM_FFN_LAG=$lag FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 256 2>&1 | tail -1)" >> $O/ab.txt
done; done
for lag in 5 6; do
  VMM_FFN_LAG=$lag FFN_MODES=fused timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:ffn_pair -s 2 -c 1 --csv python tools/bench_ffn.py 1216 256 > $O/ncu_lag$lag.csv 2>&1
  echo "lag=$lag traffic $(grep -E 'dram__bytes' $O/ncu_lag$lag.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')" >> $O/ab.txt
done
cat $O/ab.txt
