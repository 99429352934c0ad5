#!/bin/bash
O=gpurun_out/probe28; mkdir -p $O
timeout 900 python -m pytest -q -x tests/test_gpu_moe_kernels.py -k "decode_glue" tests/test_gpu_stack.py -k "decode or glue" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
timeout 900 python -m pytest -q -x tests/test_gpu_stack.py > $O/tests_stack.txt 2>&1; tail -2 $O/tests_stack.txt
timeout 900 python tools/bench_decode.py c3_qwen3vl 24 oracle,none trace > $O/decode_trace.txt 2>&1; tail -1 $O/decode_trace.txt | cut -c1-420
timeout 800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_decode.csv python tools/profile_decode.py c3_qwen3vl 4 oracle > $O/log.txt 2>&1
python tools/summarize_launches.py $O/launches_decode.csv 2>&1 | grep -E "decode_glue|skinny"
