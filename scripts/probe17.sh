timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -2 gpurun_out/pytest_gpu.log
P="timeout 200 python scripts/perf_probe.py"
for d in 0 2; do CY_DEBUG_MODE=$d $P --cfgs 5,0 --dist zeros --iters 300 --k 1024; done
for d in 0 2; do CY_DEBUG_MODE=$d $P --cfgs 5 --dist zeros --iters 300; done
$P --cfgs 5,0 --iters 1000 --torch
B="timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e"
for w in gemm dual rowreduce; do
  $B --workload $w | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['unit'], 'ms', d['ms_per_step'], d['config']['kernel_config'], 'clk', d['clocks']['sm_mhz'])"
done
