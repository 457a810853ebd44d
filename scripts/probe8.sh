timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?"; tail -3 gpurun_out/pytest_gpu.log
P="timeout 200 python scripts/perf_probe.py"
for s in 1 0; do
 echo "== sched $s"
 CY_SCHED=$s $P --cfgs 5,0 --iters 1000
 CY_SCHED=$s $P --cfgs 5,0 --iters 40 --n 16384
 CY_SCHED=$s $P --cfgs 5,0 --dist zeros --iters 300
 M="dram__bytes_read.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
 for n in 8192 16384; do
  CY_SCHED=$s timeout 120 ncu --metrics $M --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 5 --iters 2 --n $n 2>&1 | grep -E "dram__|gpu__time|lts__t_bytes|tensor"
 done
done
