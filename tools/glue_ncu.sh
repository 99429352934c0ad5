set -x
O=gpurun_out/glue
mkdir -p $O
python tools/bench_glue.py 311296 > $O/glue.log 2>&1
for k in plan_scatter combine_kernel rmsnorm_warp route_sm100; do
  case $k in plan_scatter) g=permute;; combine_kernel) g=combine;; rmsnorm_warp) g=rmsnorm;; route_sm100) g=route;; esac
  GLUE_ONLY=$g timeout 300 ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -o $O/ncu_$g python tools/bench_glue.py 311296 > $O/ncu_$g.log 2>&1
done
ls $O
