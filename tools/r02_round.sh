#!/bin/bash
# Round-2 measurement bundle (run under gpurun): GPU tests, the default bench line,
# the reference arm, R=1 lines and an ncu launch list of the bench command.
O=gpurun_out/r02
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 600 python bench.py --impl reference > $O/bench_reference.log 2>&1
timeout 600 python bench.py --requests 1 --no-cpu-baseline > $O/bench_c3_R1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
python tools/summarize_launches.py $O/launches_bench.csv > $O/launches_bench_summary.txt 2>&1
ls -la $O
