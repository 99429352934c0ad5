#!/bin/bash
# Run the R=8 headline parity test under each feature knob (one process each).
O=gpurun_out/bisect
mkdir -p $O
T="tests/test_gpu_headline.py::test_headline_shape_live_gate_decisions_and_hidden_states[8]"
for knob in NONE VMM_FFN_NO_DISCARD VMM_PREFIX_ONE_STREAM VMM_PREFIX_FULL_LAST VMM_NO_EARLY_DECIDE VMM_FFN_NO_PAIR \
            VMM_FFN_FENCE VMM_ROUTE_NO_SPLITK; do
  if [ $knob = NONE ]; then env=""; else env="$knob=1"; fi
  env $env timeout 300 python -m pytest -q -x "$T" > $O/$knob.log 2>&1
  echo "$knob exit $?" >> $O/summary.txt
done
cat $O/summary.txt
