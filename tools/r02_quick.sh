#!/bin/bash
mkdir -p gpurun_out/quick
timeout 500 python bench.py --requests 1 --workload c1_tiny --routing trace --no-cpu-baseline --steps 3 > gpurun_out/quick/c1.log 2>&1
tail -3 gpurun_out/quick/c1.log | cut -c1-600
