#!/bin/bash
# prefix: two request-aligned halves on two streams vs one stream
O=gpurun_out/probe29; mkdir -p $O
for rep in 1 2; do
  echo "two-lane: $(timeout 600 python tools/timeline_step.py 256 c3_qwen3vl 2 2>&1 | grep -E '^R=|^prefix' | tr '\n' ' ')" >> $O/p.txt
  echo "one-stream: $(VMM_PREFIX_ONE_STREAM=1 timeout 600 python tools/timeline_step.py 256 c3_qwen3vl 2 2>&1 | grep -E '^R=|^prefix' | tr '\n' ' ')" >> $O/p.txt
done
cat $O/p.txt
