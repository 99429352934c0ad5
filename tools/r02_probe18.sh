#!/bin/bash
O=gpurun_out/probe18; mkdir -p $O
for c in 1 2 4 8 16; do echo "C=$c $(VMM_PRUNE_CLUSTER=$c timeout 120 python tools/bench_prune.py 1 | tail -1)"; done > $O/prune_cluster.txt 2>&1
cat $O/prune_cluster.txt
