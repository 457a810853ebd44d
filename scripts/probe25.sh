timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -3 gpurun_out/pytest_gpu.log
B="timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e"
for w in glu dual; do
  $B --workload $w | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['unit'], d['config']['kernel_config'], 'clk', d['clocks']['sm_mhz'])"
done
