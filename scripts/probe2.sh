P="timeout 120 python scripts/perf_probe.py"
for g in 4 8 16 32; do
  echo "== group_m $g"
  CY_GROUP_M=$g $P --cfgs 0 --dist zeros --iters 200
  CY_GROUP_M=$g $P --cfgs 0 --iters 300
  CY_GROUP_M=$g $P --cfgs 0 --iters 30 --n 16384
  CY_GROUP_M=$g timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 0 --iters 2 2>&1 | grep -E "dram__|gpu__time|hit_rate"
  CY_GROUP_M=$g timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 0 --iters 2 --n 16384 2>&1 | grep -E "dram__|gpu__time"
done
