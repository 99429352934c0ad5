#!/bin/bash
O=gpurun_out/probe19; mkdir -p $O
timeout 1200 python -m pytest -q -x tests/test_gpu_headline.py -k named > $O/tests.txt 2>&1; tail -25 $O/tests.txt
