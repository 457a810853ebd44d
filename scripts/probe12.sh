timeout 600 ncu --set full --import-source on --clock-control none -k regex:cy_sm100 -s 3 -c 1 -o gpurun_out/prof_cfg5_zeros python scripts/perf_probe.py --cfgs 5 --iters 2 --dist zeros > /dev/null 2>&1; echo ncu=$?
P="timeout 200 python scripts/perf_probe.py"
for k in 1024 2048 8192; do for d in 0 2; do CY_DEBUG_MODE=$d $P --cfgs 5,0 --dist zeros --iters 300 --k $k; done; done
