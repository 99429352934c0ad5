#!/bin/bash
O=gpurun_out/r02h; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 600 python bench.py --impl reference > $O/bench_reference.log 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
tail -1 $O/bench_default.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), round(d["e2e"]["serial"]["value"]), d["clocks"])'
tail -1 $O/bench_reference.log | cut -c1-200
