P="timeout 200 python scripts/perf_probe.py"
for d in 0 2 4 8; do CY_DEBUG_MODE=$d $P --cfgs 5,0 --dist zeros --iters 300 --k 1024; done
