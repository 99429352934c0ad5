#!/bin/bash
O=gpurun_out/probe15; mkdir -p $O
for rep in 1 2; do timeout 120 python tools/bench_skinny.py 8 >> $O/skinny.txt 2>&1; done
timeout 120 python tools/bench_skinny.py 16 >> $O/skinny.txt 2>&1
timeout 120 python tools/bench_skinny.py 1 >> $O/skinny.txt 2>&1
cat $O/skinny.txt
timeout 900 python -m pytest -q -x tests/test_gpu_moe_kernels.py tests/test_gpu_stack.py tests/test_gpu_headline.py > $O/tests.txt 2>&1; tail -2 $O/tests.txt
timeout 900 python tools/bench_decode.py c3_qwen3vl 24 oracle,none trace > $O/decode_trace.txt 2>&1; tail -1 $O/decode_trace.txt | cut -c1-500
