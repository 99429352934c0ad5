#!/bin/bash
O=gpurun_out/probe11; mkdir -p $O
timeout 900 python -m pytest -q -x tests/test_gpu_moe_kernels.py tests/test_gpu_stack.py -k "skinny or router or decode or route" > $O/tests.txt 2>&1; tail -3 $O/tests.txt
VMM_ROUTE_SPLIT=0 timeout 300 python tools/route_split_sweep.py child > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 900 python tools/bench_decode.py c3_qwen3vl 24 gate,history,none live > $O/decode_live.txt 2>&1; tail -1 $O/decode_live.txt | cut -c1-1500
