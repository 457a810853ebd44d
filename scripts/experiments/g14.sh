timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/g14_pytest.txt 2>&1; echo "pytest=$?"; tail -3 gpurun_out/g14_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g14_smoke.txt 2>&1; echo "smoke=$?"; tail -1 gpurun_out/g14_smoke.txt
timeout 600 python bench.py > gpurun_out/g14_bench.json 2> gpurun_out/g14_bench.err; echo "bench=$?"; cat gpurun_out/g14_bench.json
