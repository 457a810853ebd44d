set -u
timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q -k "splitk" > gpurun_out/g9_splitk.txt 2>&1; echo "splitk=$?"; tail -15 gpurun_out/g9_splitk.txt
timeout 600 python scripts/splitk_probe.py > gpurun_out/g9_probe.txt 2>&1; echo "probe=$?"; cat gpurun_out/g9_probe.txt
