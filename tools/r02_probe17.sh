#!/bin/bash
O=gpurun_out/probe17; mkdir -p $O
timeout 600 python -m pytest -q -x tests/test_gpu_moe_kernels.py -k "rout" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
for mc in 1 2 4; do
  echo "MC=$mc" >> $O/times.txt
  VMM_ROUTE_MC=$mc timeout 300 python tools/route_big.py 311296 7 >> $O/times.txt 2>&1
  VMM_ROUTE_MC=$mc timeout 300 python tools/route_big.py 606208 5 >> $O/times.txt 2>&1
  VMM_ROUTE_MC=$mc timeout 300 python tools/route_big.py 9728 9 >> $O/times.txt 2>&1
done
cat $O/times.txt
timeout 900 python -m pytest -q -x tests/test_gpu_headline.py tests/test_gpu_stack.py > $O/tests2.txt 2>&1; tail -2 $O/tests2.txt
