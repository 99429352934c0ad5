#!/bin/bash
# variance check: the default bench with 20 timed steps, twice, and the reference arm with 10
O=gpurun_out/long; mkdir -p $O
timeout 1500 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench20_a.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench20_b.log 2>&1
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > $O/ref10.log 2>&1
for f in $O/bench20_a.log $O/bench20_b.log; do tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), round(d["ms_per_step"],1), d["clocks"])'; done
tail -1 $O/ref10.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("ref", round(d["value"]), round(d["ms_per_step"],1))'
