set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/r2b_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r2b_bench_c4.json 2> gpurun_out/r2b_bench_c4.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.txt 2>&1; echo "exit $?" >> gpurun_out/r2b_smoke.txt
