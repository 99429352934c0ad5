#!/bin/bash
# Round-end measurement bundle (run under gpurun): bench lines for every config,
# the reference arm, an ncu launch list of one R=256 step and a full capture of the FFN.
set -x
mkdir -p gpurun_out/round
O=gpurun_out/round
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 300 python bench.py --impl reference > $O/bench_reference.log 2>&1
timeout 600 python bench.py --requests 1 --no-cpu-baseline > $O/bench_c3_R1.log 2>&1
timeout 600 python bench.py --requests 1 --workload c2_phi2 --no-cpu-baseline > $O/bench_c2_R1.log 2>&1
timeout 600 python bench.py --requests 1 --workload c4_dsvl2s --no-cpu-baseline > $O/bench_c4_R1.log 2>&1
timeout 600 python bench.py --requests 1 --workload c1_tiny --routing trace --no-cpu-baseline > $O/bench_c1_R1.log 2>&1
timeout 600 python bench.py --requests 1 --source sharded --no-cpu-baseline > $O/bench_c3_R1_sharded.log 2>&1
VMM_FFN_FENCE=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches_R256.csv python tools/timeline_step.py 256 c3_qwen3vl 1 > $O/ncu_tl.log 2>&1
python tools/summarize_launches.py $O/launches_R256.csv > $O/launches_R256_summary.txt 2>&1
FFN_MODES=fused timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_pair -s 2 -c 1 \
  -o $O/ncu_ffn_pair_R256 python tools/bench_ffn.py 1216 256 > $O/ncu_ffn.log 2>&1
ls -la $O
