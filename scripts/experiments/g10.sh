timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q -k "splitk" > gpurun_out/g10.txt 2>&1; echo "rc=$?"; tail -5 gpurun_out/g10.txt
