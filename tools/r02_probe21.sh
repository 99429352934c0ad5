#!/bin/bash
O=gpurun_out/probe21; mkdir -p $O
timeout 600 python bench.py --requests 8 --no-cpu-baseline > $O/r8.log 2>&1; tail -c 700 $O/r8.log; echo
timeout 900 python bench.py --no-cpu-baseline > $O/r256.log 2>&1; tail -1 $O/r256.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["e2e"]["value"], d["e2e"]["ms_per_step"], d["e2e"]["serial"], d["ms_per_step"])'
timeout 600 python bench.py --requests 1 --no-cpu-baseline > $O/r1.log 2>&1; tail -1 $O/r1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["e2e"]["value"], d["e2e"]["serial"]["value"])'
