#!/bin/bash
O=gpurun_out/probe14; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:skinny_ffn -s 3 -c 1 \
  -o $O/ncu_skinny python tools/bench_skinny.py 8 > $O/ncu.log 2>&1
ls $O
