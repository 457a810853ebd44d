P="timeout 200 python scripts/perf_probe.py"
M="dram__bytes_read.sum,gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_requests_srcunit_tex.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for pr in 3 2 0; do
 echo "== promo $pr"
 CY_L2_PROMO=$pr $P --cfgs 5 --iters 1000
 CY_L2_PROMO=$pr timeout 120 ncu --metrics $M --clock-control none -k regex:cy_sm100 -s 5 -c 1 python scripts/perf_probe.py --cfgs 5 --iters 2 2>&1 | grep -E "dram__|gpu__time|lts__|tensor"
done
echo "== cublas"
timeout 120 ncu --metrics $M --clock-control none -s 4 -c 1 python scripts/torch_mm.py 8192 2>&1 | grep -E "dram__|gpu__time|lts__|tensor"
echo "== epilogue exposure cfg5/cfg0 zeros"
for d in 0 2; do CY_DEBUG_MODE=$d $P --cfgs 5,0 --dist zeros --iters 300; done
