#!/bin/bash
# router split sweep + FFN DRAM traffic with / without the H1 discard
O=gpurun_out/probe1
mkdir -p $O
timeout 600 python tools/route_split_sweep.py > $O/route_split.txt 2>&1
for d in 0 1; do
  if [ $d = 1 ]; then export VMM_FFN_NO_DISCARD=1; else unset VMM_FFN_NO_DISCARD; fi
  FFN_MODES=fused timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum \
    --clock-control none -k regex:ffn_pair -c 3 --csv python tools/bench_ffn.py 1216 256 > $O/ffn_traffic_nodiscard$d.csv 2>&1
  FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 256 > $O/ffn_time_nodiscard$d.txt 2>&1
done
unset VMM_FFN_NO_DISCARD
timeout 600 python -m pytest -q tests/test_gpu_moe_kernels.py > $O/moe_kernels.log 2>&1
tail -3 $O/moe_kernels.log
cat $O/route_split.txt $O/ffn_time_nodiscard*.txt
