#!/bin/bash
O=gpurun_out/probe30; mkdir -p $O
for rep in 1 2 3; do
  echo "byvalue $(timeout 600 python tools/bench_decode.py c3_qwen3vl 24 oracle trace 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["oracle"]["decode_tokens_per_s"],1))')" >> $O/ab.txt
  echo "upload  $(VMM_DECODE_UPLOAD_ROWS=1 timeout 600 python tools/bench_decode.py c3_qwen3vl 24 oracle trace 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["oracle"]["decode_tokens_per_s"],1))')" >> $O/ab.txt
done
cat $O/ab.txt
