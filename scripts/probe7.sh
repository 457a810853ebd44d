timeout 300 python scripts/quick_check.py 5 2>&1 | grep -v "^n=" 
P="timeout 200 python scripts/perf_probe.py"
$P --cfgs 0,5 --iters 1000 --torch
$P --cfgs 0,5 --dist zeros --iters 300
$P --cfgs 0,5 --iters 40 --n 16384 --torch
$P --cfgs 0,5 --iters 1000 --n 4096
M="dram__bytes_read.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for n in 8192 16384; do
CY_GROUP_M=8 timeout 120 ncu --metrics $M --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 5 --iters 2 --n $n 2>&1 | grep -E "dram__|gpu__time|lts__t_bytes|tensor"
done
