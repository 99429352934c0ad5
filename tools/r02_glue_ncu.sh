#!/bin/bash
# round-2 ncu --set full captures of the R=256 glue kernels and the batched prune
O=gpurun_out/glue2; mkdir -p $O
python tools/bench_glue.py 311296 > $O/glue.log 2>&1
for k in plan_scatter combine_kernel rmsnorm_warp; do
  case $k in plan_scatter) g=permute;; combine_kernel) g=combine;; rmsnorm_warp) g=rmsnorm;; esac
  GLUE_ONLY=$g timeout 300 ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -o $O/ncu_$g python tools/bench_glue.py 311296 > $O/ncu_$g.log 2>&1
done
timeout 300 ncu --set full --clock-control none -k regex:prune -s 5 -c 1 -o $O/ncu_prune_R256 python tools/bench_prune.py 256 > $O/ncu_prune.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:prune -s 5 -c 1 -o $O/ncu_prune_R1 python tools/bench_prune.py 1 > $O/ncu_prune1.log 2>&1
ls $O; cat $O/glue.log
