# Round-end GPU refresh (run under gpurun from the repo root): full parity suite, smoke, every
# bench workload, the ncu launch list of the headline bench and one ncu --set full capture per
# dominant kernel.  Outputs land in gpurun_out/ (copy the summaries into profiles/).
set -u
R=${ROUND:-r01}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_exit=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench_exit=$?"; cat gpurun_out/bench_default.json
for w in batched dual glu rowreduce attention sweep-1024 sweep-2048 sweep-4096 sweep-16384; do
  timeout 900 python bench.py --workload $w --steps 300 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w exit=$?"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${R}_gemm.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_list=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_${R}_attention.csv \
  python bench.py --workload attention --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_list_attn=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cy_sm100 -s 3 -c 1 -f -o gpurun_out/prof_${R}_gemm \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_full=$?"
for w in batched dual rowreduce; do
  timeout 600 ncu --set full --clock-control none -k regex:cy_sm100 -s 3 -c 1 -f -o gpurun_out/prof_${R}_$w \
    python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_$w=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 -f -o gpurun_out/prof_${R}_attention \
  python bench.py --workload attention --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_attn=$?"
