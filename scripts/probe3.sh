P="timeout 120 python scripts/perf_probe.py"
for pol in 0 1 2 3 4 5; do
  echo "== l2 policy $pol"
  CY_L2_POLICY=$pol $P --cfgs 0 --iters 300
  CY_L2_POLICY=$pol $P --cfgs 0 --iters 30 --n 16384
  CY_L2_POLICY=$pol timeout 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 0 --iters 2 2>&1 | grep -E "dram__|gpu__time|hit_rate"
  CY_L2_POLICY=$pol timeout 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 0 --iters 2 --n 16384 2>&1 | grep -E "dram__|gpu__time"
done
timeout 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -s 5 -c 1 python scripts/perf_probe.py --cfgs 0 --iters 2 --torch 2>&1 | grep -E "dram__|gpu__time|Kernel|void|sm100"
timeout 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -s 5 -c 1 python scripts/perf_probe.py --cfgs 0 --iters 2 --torch --n 16384 2>&1 | grep -E "dram__|gpu__time|Kernel|void|sm100"
