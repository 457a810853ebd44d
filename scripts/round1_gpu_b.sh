timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench_exit=$?"; cat gpurun_out/bench_default.json
for w in batched dual rowreduce sweep-1024 sweep-2048 sweep-4096 sweep-16384; do
  timeout 600 python bench.py --workload $w --steps 300 --no-cpu-baseline > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; echo "$w exit=$?"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_list=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cy_sm100 -s 3 -c 1 -o gpurun_out/prof_r01b_gemm8192 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_full=$?"
for w in batched dual rowreduce; do
timeout 600 ncu --set full --clock-control none -k regex:cy_sm100 -s 3 -c 1 -o gpurun_out/prof_r01b_$w python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_$w=$?"
done
