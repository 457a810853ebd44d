set -u
for g in 8 12 16 6 24 4; do
  echo "g=$g" >> gpurun_out/g7_bench.txt
  CY_GROUP_M=$g timeout 300 python bench.py --steps 2500 --warmup 20 --no-cpu-baseline --no-e2e >> gpurun_out/g7_bench.txt 2>&1
  CY_GROUP_M=$g timeout 300 python bench.py --workload rowreduce --steps 250 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/g7_bench.txt 2>&1
  CY_GROUP_M=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cy_sm100 -s 5 -c 2 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g7_ncu_g$g.csv 2>/dev/null
  CY_GROUP_M=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cy_sm100 -s 5 -c 2 --csv python bench.py --workload rowreduce --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g7_ncu_rr_g$g.csv 2>/dev/null
done
echo done
