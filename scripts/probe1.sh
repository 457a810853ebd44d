set -x
P="timeout 120 python scripts/perf_probe.py"
$P --cfgs 0,2 --torch --iters 100
$P --cfgs 0 --torch --iters 1000
$P --cfgs 0 --torch --dist zeros --iters 200
$P --cfgs 0 --torch --dist randn --iters 200
$P --cfgs 0 --k 4096 --iters 200
$P --cfgs 0 --k 16384 --iters 100
$P --cfgs 0 --torch --n 4096 --iters 300
$P --cfgs 0,1,2,3,4 --torch --n 2048 --iters 500
$P --cfgs 0,1,2,3,4 --torch --n 1024 --iters 1000
$P --cfgs 0 --torch --n 16384 --iters 20
