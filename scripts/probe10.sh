B="timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e"
for w in sweep-1024 sweep-2048 sweep-4096 gemm sweep-16384 batched dual rowreduce; do
  $B --workload $w | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['unit'], 'ms', d['ms_per_step'], d['config']['kernel_config'], 'clk', d['clocks']['sm_mhz'])"
done
P="timeout 200 python scripts/perf_probe.py --torch"
$P --cfgs 0 --n 1024 --iters 2000
$P --cfgs 0 --n 2048 --iters 1000
