#!/bin/bash
O=gpurun_out/probe13; mkdir -p $O
timeout 300 python tools/route_big.py 311296 7 > $O/times.txt 2>&1; cat $O/times.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_sm100 -s 1 -c 1 \
  -o $O/ncu_route1 python tools/route_big.py 311296 2 > $O/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_sm100 -s 3 -c 1 \
  -o $O/ncu_route2 python tools/route_big.py 311296 2 > $O/ncu2.log 2>&1
ls $O
