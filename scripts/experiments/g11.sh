timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q -k "splitk" > gpurun_out/g11.txt 2>&1; echo "rc=$?"; tail -5 gpurun_out/g11.txt
timeout 600 python scripts/splitk_probe.py > gpurun_out/g11_probe.txt 2>&1; cat gpurun_out/g11_probe.txt
