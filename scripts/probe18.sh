P="timeout 200 python scripts/perf_probe.py"
$P --cfgs 0,1,5 --dist zeros --iters 300 --k 1024
$P --cfgs 0,5 --dist zeros --iters 300
$P --cfgs 0,2,3 --iters 300 --n 4096
B="timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for w in batched sweep-2048 sweep-4096; do
  $B --workload $w | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['unit'], 'ms', d['ms_per_step'], d['config']['kernel_config'], 'clk', d['clocks']['sm_mhz'])"
done
