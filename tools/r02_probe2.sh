#!/bin/bash
# FFN DRAM traffic / time vs L2 store hints and GEMM2 lag (discard on)
O=gpurun_out/probe2
mkdir -p $O
for lag in 4 2 8; do for h in 0 1 2 3; do
  VMM_FFN_LAG=$lag VMM_FFN_L2HINTS=$h FFN_MODES=fused timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:ffn_pair -s 2 -c 1 --csv python tools/bench_ffn.py 1216 256 > $O/ncu_lag${lag}_h$h.csv 2>&1
  VMM_FFN_LAG=$lag VMM_FFN_L2HINTS=$h FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 256 > $O/time_lag${lag}_h$h.txt 2>&1
  r=$(grep dram__bytes_read $O/ncu_lag${lag}_h$h.csv | awk -F'","' '{print $NF}' | tr -d '"')
  w=$(grep dram__bytes_write $O/ncu_lag${lag}_h$h.csv | awk -F'","' '{print $NF}' | tr -d '"')
  echo "lag=$lag hints=$h read=$r write=$w $(cat $O/time_lag${lag}_h$h.txt | tail -1)" >> $O/summary.txt
done; done
cat $O/summary.txt
