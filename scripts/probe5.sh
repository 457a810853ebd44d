P="timeout 120 python scripts/perf_probe.py"
for d in 0 1 2 3; do
  echo "== debug $d"
  CY_DEBUG_MODE=$d $P --cfgs 0,2 --dist zeros --iters 200
  CY_DEBUG_MODE=$d $P --cfgs 0 --dist zeros --iters 50 --n 16384
  CY_DEBUG_MODE=$d $P --cfgs 0 --dist zeros --iters 200 --k 16384
done
