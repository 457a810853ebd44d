timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q -k "splitk" > gpurun_out/g13.txt 2>&1; echo "rc=$?"; tail -3 gpurun_out/g13.txt
timeout 800 python scripts/splitk_grid.py > gpurun_out/g13_grid.txt 2>&1; grep -v "^   c" gpurun_out/g13_grid.txt
