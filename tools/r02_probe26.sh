#!/bin/bash
# FFN tile schedule A/B: per-cluster m-tiles (sched 1) vs global block order (sched 0)
O=gpurun_out/probe26; mkdir -p $O
timeout 900 python -m pytest -q -x tests/test_gpu_moe_kernels.py -k "fused_ffn" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
for rep in 1 2 3 4; do for sc in 1 0; do
  echo "rep=$rep sched=$sc $(VMM_FFN_SCHED=$sc FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 256 2>&1 | tail -1)" >> $O/ab.txt
done; done
echo "R=64 rows:" >> $O/ab.txt
for sc in 1 0; do echo "sched=$sc $(VMM_FFN_SCHED=$sc FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 64 2>&1 | tail -1)" >> $O/ab.txt; done
cat $O/ab.txt
VMM_LIB=$PWD/paper_2605_05899_b200/libvismmoe_prof.so timeout 300 python tools/ffn_prof.py 1216 256 > $O/prof1.txt 2>&1
VMM_FFN_SCHED=0 VMM_LIB=$PWD/paper_2605_05899_b200/libvismmoe_prof.so timeout 300 python tools/ffn_prof.py 1216 256 > $O/prof0.txt 2>&1
grep -E "not ready|flag/H1|MMA busy|full wait" $O/prof1.txt $O/prof0.txt
FFN_MODES=fused timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:ffn_pair -s 2 -c 1 --csv python tools/bench_ffn.py 1216 256 > $O/ncu1.csv 2>&1
grep -E "dram__bytes|gpu__time" $O/ncu1.csv | awk -F'","' '{print $(NF-2), $NF}'
