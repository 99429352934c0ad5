#!/bin/bash
O=gpurun_out/probe27; mkdir -p $O
for c in 0 12288 6144 24576; do echo "chunk=$c $(VMM_COMBINE_CHUNK=$c GLUE_ONLY=combine_norm timeout 200 python tools/bench_glue.py 311296 | grep combine_norm)"; done > $O/cn.txt 2>&1
for c in 0 6144; do echo "rep2 chunk=$c $(VMM_COMBINE_CHUNK=$c GLUE_ONLY=combine_norm timeout 200 python tools/bench_glue.py 311296 | grep combine_norm)"; done >> $O/cn.txt 2>&1
cat $O/cn.txt
timeout 600 python -m pytest -q -x tests/test_gpu_moe_kernels.py -k "combine" tests/test_gpu_stack.py > $O/tests.txt 2>&1; tail -2 $O/tests.txt
