#!/bin/bash
# walk order: parity tests, timeline and bench A/B
O=gpurun_out/probe9; mkdir -p $O
timeout 900 python -m pytest -q -x tests/test_gpu_moe_kernels.py tests/test_gpu_headline.py tests/test_gpu_stack.py > $O/tests.txt 2>&1; tail -3 $O/tests.txt
timeout 500 python tools/timeline_step.py 256 c3_qwen3vl 3 > $O/tl.txt 2>&1; head -8 $O/tl.txt
for rep in 1 2; do
timeout 900 python bench.py --no-cpu-baseline > $O/bench_walk_$rep.log 2>&1
VMM_NO_WALK_ORDER=1 timeout 900 python bench.py --no-cpu-baseline > $O/bench_nowalk_$rep.log 2>&1
done
for f in $O/bench_*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), round(d["ms_per_step"],1), d["clocks"]["sm_mhz"])')"; done
