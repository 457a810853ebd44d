# Round-end GPU refresh (run under gpurun from the repo root): full parity suite, smoke, every
# bench workload, the ncu launch list of the headline bench and one ncu --set full capture per
# dominant kernel.  Outputs land in gpurun_out/ (copy the summaries into profiles/).
set -u
R=${ROUND:-r02d}
mkdir -p gpurun_out/$R
O=gpurun_out/$R
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_exit=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench_exit=$?"; cat $O/bench_default.json
timeout 900 python bench.py --steps 3000 --warmup 20 --no-cpu-baseline --no-e2e > $O/bench_sustained.json 2>&1; echo "sustained=$?"
for w in batched batched-beta1 dual glu rowreduce attention sweep-1024 sweep-2048 sweep-4096 sweep-16384 allgather allgather-fused; do
  timeout 900 python bench.py --workload $w --steps 300 > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w exit=$?"
done
for w in sweep-1024 sweep-2048 sweep-4096; do
  timeout 600 python bench.py --workload $w --steps 200 --graph --no-cpu-baseline --no-e2e > $O/bench_${w}_graph.json 2>&1; echo "$w graph exit=$?"
done
timeout 600 python scripts/splitk_grid.py > $O/splitk_grid.txt 2>&1; echo "splitk_grid=$?"
timeout 600 python scripts/sweep_vs_cublas.py > $O/sweep_vs_cublas.txt 2>&1; echo "sweep=$?"
timeout 600 python scripts/batched_cfg_sweep.py 64 400 > $O/batched_cfg.txt 2>&1; echo "batched_cfg=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_${R}_gemm.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_list=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_${R}_attention.csv \
  python bench.py --workload attention --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_list_attn=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cy_sm100 -s 3 -c 1 -f -o $O/prof_${R}_gemm \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_full=$?"
for w in batched dual rowreduce; do
  timeout 600 ncu --set full --clock-control none -k regex:cy_sm100 -s 3 -c 1 -f -o $O/prof_${R}_$w \
    python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_$w=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 -f -o $O/prof_${R}_attention \
  python bench.py --workload attention --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_attn=$?"
timeout 600 python scripts/attn_probe.py > $O/attn_probe.txt 2>&1; echo "attn_probe=$?"
# summaries on the box; keep only the headline GEMM and attention reports (gpurun copies back <= 64 MiB)
python scripts/ncu_summary.py gemm=$O/prof_${R}_gemm.ncu-rep batched=$O/prof_${R}_batched.ncu-rep dual=$O/prof_${R}_dual.ncu-rep \
  rowreduce=$O/prof_${R}_rowreduce.ncu-rep attention=$O/prof_${R}_attention.ncu-rep > $O/ncu_summary.json 2>&1; echo "ncu_summary=$?"
rm -f $O/prof_${R}_batched.ncu-rep $O/prof_${R}_dual.ncu-rep $O/prof_${R}_rowreduce.ncu-rep
