#!/bin/bash
O=gpurun_out/probe12; mkdir -p $O
for rep in 1 2; do
  timeout 120 python tools/bench_skinny.py 8 >> $O/skinny.txt 2>&1
  VMM_SKINNY_NO_PF=1 timeout 120 python tools/bench_skinny.py 8 | sed 's/^/nopf /' >> $O/skinny.txt 2>&1
done
cat $O/skinny.txt
timeout 600 python -m pytest -q -x tests/test_gpu_moe_kernels.py tests/test_gpu_stack.py -k "decode or skinny or waits" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
timeout 900 python tools/bench_decode.py c3_qwen3vl 24 oracle trace > $O/decode_trace.txt 2>&1; tail -1 $O/decode_trace.txt | cut -c1-400
VMM_SKINNY_NO_PF=1 timeout 900 python tools/bench_decode.py c3_qwen3vl 24 oracle trace > $O/decode_trace_nopf.txt 2>&1; tail -1 $O/decode_trace_nopf.txt | cut -c1-400
