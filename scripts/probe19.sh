timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -2 gpurun_out/pytest_gpu.log
for pdl in 0 1; do echo "== pdl $pdl"; CY_PDL=$pdl timeout 300 python scripts/latency_probe.py 2>&1 | grep ours; done
B="timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for w in batched sweep-1024 sweep-2048; do
  $B --workload $w | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['unit'], 'ms', d['ms_per_step'], d['config']['kernel_config'], 'clk', d['clocks']['sm_mhz'])"
done
