#!/bin/bash
# FFN A/B: round-2 default (discard + L2 hints) vs round-1 behaviour (no discard, no hints), alternating
O=gpurun_out/probe23; mkdir -p $O
for rep in 1 2 3 4; do
  echo "rep=$rep new $(FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 256 2>&1 | tail -1)" >> $O/ab.txt
  echo "rep=$rep old $(VMM_FFN_NO_DISCARD=1 VMM_FFN_L2HINTS=0 FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 256 2>&1 | tail -1)" >> $O/ab.txt
  echo "rep=$rep nodiscard_hints $(VMM_FFN_NO_DISCARD=1 FFN_MODES=fused timeout 300 python tools/bench_ffn.py 1216 256 2>&1 | tail -1)" >> $O/ab.txt
done
cat $O/ab.txt
