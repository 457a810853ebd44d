timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/g15_pytest.txt 2>&1; echo "pytest=$?"; tail -3 gpurun_out/g15_pytest.txt; grep FAILED gpurun_out/g15_pytest.txt | head
