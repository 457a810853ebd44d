for L in 8 64; do for c in 0 5 2; do timeout 100 python scripts/batched_probe.py $L $c 300 2>&1 | grep "cfg"; done; timeout 100 python scripts/batched_probe.py $L -1 300 2>&1 | grep bmm; done
timeout 300 ncu --set full --clock-control none -k regex:cy_sm100 -s 12 -c 1 -o gpurun_out/prof_b8 python scripts/batched_probe.py 8 5 3 > /dev/null 2>&1; echo ncu=$?
