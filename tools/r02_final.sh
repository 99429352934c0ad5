#!/bin/bash
# Final round-2 bundle: GPU tests, smoke, every bench line, the reference arm, an ncu launch
# list of the default bench command and a full capture of the FFN.
O=gpurun_out/r02f
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 600 python bench.py --impl reference > $O/bench_reference.log 2>&1
timeout 600 python bench.py --requests 1 --no-cpu-baseline > $O/bench_c3_R1.log 2>&1
timeout 600 python bench.py --requests 8 --no-cpu-baseline > $O/bench_c3_R8.log 2>&1
timeout 600 python bench.py --requests 1 --workload c2_phi2 --no-cpu-baseline > $O/bench_c2_R1.log 2>&1
timeout 600 python bench.py --requests 1 --workload c4_dsvl2s --no-cpu-baseline > $O/bench_c4_R1.log 2>&1
timeout 600 python bench.py --requests 1 --workload c1_tiny --routing trace --no-cpu-baseline > $O/bench_c1_R1.log 2>&1
timeout 600 python bench.py --requests 1 --source sharded --no-cpu-baseline > $O/bench_c3_R1_sharded.log 2>&1
timeout 900 python bench.py --source sharded --no-cpu-baseline > $O/bench_c3_R256_sharded.log 2>&1
VMM_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --requests 16 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_share2_R16.log 2>&1
timeout 900 python tools/bench_decode.py c3_qwen3vl 24 oracle,none trace > $O/decode_trace.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
python tools/summarize_launches.py $O/launches_bench.csv > $O/launches_bench_summary.txt 2>&1
FFN_MODES=fused timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_pair -s 2 -c 1 \
  -o $O/ncu_ffn_pair_R256 python tools/bench_ffn.py 1216 256 > $O/ncu_ffn.log 2>&1
ls -la $O
