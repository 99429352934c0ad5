#!/bin/bash
# compute-sanitizer racecheck / memcheck on the copy-overlapped FFN (CTA-pair path, H1 discard,
# walk order) and a tiny stack forward with live routing
O=gpurun_out/sanitize; mkdir -p $O
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x \
  "tests/test_gpu_moe_kernels.py::test_fused_ffn_waits_for_copy_stream_fills[5000]" \
  "tests/test_gpu_moe_kernels.py::test_router_chunks_bit_identical_to_one_launch" > $O/memcheck.log 2>&1
tail -5 $O/memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -q -x \
  "tests/test_gpu_moe_kernels.py::test_fused_ffn_waits_for_copy_stream_fills[5000]" > $O/racecheck.log 2>&1
tail -5 $O/racecheck.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x tests/test_gpu_stack.py -k "live" > $O/memcheck_stack.log 2>&1
tail -5 $O/memcheck_stack.log
