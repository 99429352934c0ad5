O=gpurun_out/probe5; mkdir -p $O
timeout 600 python -m pytest -q tests/test_gpu_moe_kernels.py -k "router or route" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
export VMM_LIB=$PWD/paper_2605_05899_b200/libvismmoe_prof.so
for n in 1216 2368; do for la in 0 1; do echo "== route N=$n la=$la"; timeout 120 python tools/route_prof.py $n $la; done; done > $O/route_prof.txt 2>&1
unset VMM_LIB
timeout 300 python tools/route_split_sweep.py > $O/sweep.txt 2>&1
cat $O/route_prof.txt | grep -E "==|reduce|span"; head -2 $O/sweep.txt
