timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -2 gpurun_out/pytest_gpu.log
P="timeout 200 python scripts/perf_probe.py"
for r in 1 2; do
for ar in 0 1; do echo "== a_reuse $ar"; CY_A_REUSE=$ar $P --cfgs 5 --iters 1500; done
done
for ar in 0 1; do CY_A_REUSE=$ar $P --cfgs 5 --dist zeros --iters 300; done
$P --cfgs 5 --iters 1500 --torch
B="timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e"
for ar in 0 1; do for w in dual rowreduce; do
  CY_A_REUSE=$ar $B --workload $w | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('a_reuse $ar $w', d['value'], d['unit'], 'clk', d['clocks']['sm_mhz'])"
done; done
