#!/bin/bash
# refresh the bench lines after the streamed-e2e change (kernels unchanged since tools/r02_final.sh)
O=gpurun_out/r02g; mkdir -p $O
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
ls -la $O
