#!/bin/bash
# shared host pool: 2-process tests + a 2-rank bench on one GPU (gloo), /dev/shm capacity
O=gpurun_out/probe6; mkdir -p $O
df -h /dev/shm > $O/shm.txt; free -g >> $O/shm.txt
timeout 900 python -m pytest -q tests/test_gpu_ep.py > $O/ep_tests.txt 2>&1; tail -3 $O/ep_tests.txt
VMM_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --requests 16 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_share2.log 2>&1
tail -c 1500 $O/bench_share2.log
cat $O/shm.txt
