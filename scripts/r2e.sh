set -x
timeout 900 python -m pytest tests/test_gpu_module_full.py -q -x > gpurun_out/r2e_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/r2e_pytest.txt
