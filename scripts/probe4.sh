M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__block_size,launch__shared_mem_per_block_dynamic"
for n in 8192 16384; do
 echo "== cublas $n"
 timeout 120 ncu --metrics $M --clock-control none -s 4 -c 1 python scripts/torch_mm.py $n 2>&1 | grep -vE "^==PROF|^$" | tail -16
 echo "== ours $n"
 timeout 120 ncu --metrics $M --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 0 --iters 2 --n $n 2>&1 | grep -vE "^==PROF|^$" | tail -14
done
