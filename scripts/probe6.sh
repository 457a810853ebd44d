P="timeout 200 python scripts/perf_probe.py"
for d in 0 1 2 3; do
  echo "== debug $d"
  CY_DEBUG_MODE=$d $P --cfgs 0 --iters 1000
done
$P --cfgs 0 --iters 1000 --torch
