#!/bin/bash
O=gpurun_out/probe16; mkdir -p $O
timeout 900 python -m pytest -q -x tests/test_gpu_moe_kernels.py -k "rout" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
timeout 300 python tools/route_big.py 311296 7 > $O/times.txt 2>&1; cat $O/times.txt
timeout 300 python tools/route_big.py 606208 5 >> $O/times.txt 2>&1; tail -2 $O/times.txt
timeout 300 python tools/route_split_sweep.py child > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 900 python -m pytest -q -x tests/test_gpu_headline.py tests/test_gpu_stack.py > $O/tests2.txt 2>&1; tail -2 $O/tests2.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; tail -1 $O/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), round(d["ms_per_step"],1), d["clocks"]["sm_mhz"])'
