M="gpu__time_duration.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_bytes.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active"
for c in 4 3 0 2; do
echo "== cfg $c"
timeout 120 ncu --metrics $M --clock-control none -k regex:cy_sm100 -s 8 -c 1 python scripts/perf_probe.py --cfgs $c --iters 5 --n 1024 2>&1 | grep -E "gpu__|sm__|gpc__|dram__|lts__|launch__"
done
echo "== cublas"
timeout 120 ncu --metrics $M --clock-control none -s 6 -c 1 python scripts/torch_mm.py 1024 2>&1 | grep -E "gpu__|sm__|gpc__|dram__|lts__|launch__|Cfg|void|nvjet" 
