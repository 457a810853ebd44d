M="dram__bytes_read.sum,gpu__time_duration.sum"
for g in 4 8 16 32; do
 echo "== group_m $g"
 CY_GROUP_M=$g timeout 200 python scripts/perf_probe.py --cfgs 5 --iters 300
 CY_GROUP_M=$g timeout 200 python scripts/perf_probe.py --cfgs 5 --iters 30 --n 16384
 CY_GROUP_M=$g timeout 200 python scripts/perf_probe.py --cfgs 5 --iters 30 --m 65536 --n 8192 --k 8192
 for sh in "--n 8192" "--n 16384" "--m 65536 --n 8192 --k 8192"; do
  CY_GROUP_M=$g timeout 120 ncu --metrics $M --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 5 --iters 2 $sh 2>&1 | grep -E "dram__|gpu__time" | tr '\n' ' '; echo
 done
done
