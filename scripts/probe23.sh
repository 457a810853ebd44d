P="timeout 200 python scripts/perf_probe.py"
for r in 1 2; do
for ns in 0 256 2048; do echo "== sleep $ns"; CY_SLEEP_NS=$ns $P --cfgs 5 --iters 1500; done
done
CY_SLEEP_NS=0 $P --cfgs 5 --dist zeros --iters 300
CY_SLEEP_NS=2048 $P --cfgs 5 --dist zeros --iters 300
$P --cfgs 5 --iters 1500 --torch
