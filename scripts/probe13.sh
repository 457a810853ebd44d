timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -2 gpurun_out/pytest_gpu.log
P="timeout 200 python scripts/perf_probe.py"
for k in 1024 8192; do for d in 0 2; do CY_DEBUG_MODE=$d $P --cfgs 5,0 --dist zeros --iters 300 --k $k; done; done
$P --cfgs 5,0 --iters 1000 --torch
