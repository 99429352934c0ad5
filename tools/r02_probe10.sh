#!/bin/bash
# decode lines with the round-2 code + ncu of the decode-sized router
O=gpurun_out/probe10; mkdir -p $O
timeout 900 python tools/bench_decode.py c3_qwen3vl 24 oracle,none trace > $O/decode_trace.txt 2>&1
timeout 900 python tools/bench_decode.py c3_qwen3vl 24 gate,history,mlp,none live > $O/decode_live.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size,launch__block_size \
  --clock-control none -k regex:skinny -c 20 --csv python tools/route_split_sweep.py child > $O/ncu_skinny_route.csv 2>&1
tail -4 $O/decode_trace.txt; tail -6 $O/decode_live.txt
grep -E "skinny" $O/ncu_skinny_route.csv | head -12
