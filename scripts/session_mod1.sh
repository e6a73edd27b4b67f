set -x
timeout 240 python -m pytest tests/test_gpu_module.py -x -q > gpurun_out/m1_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/m1_pytest.txt
timeout 240 python -m pytest tests/test_gpu_module.py -q > gpurun_out/m1_pytest_all.txt 2>&1; echo "exit $?" >> gpurun_out/m1_pytest_all.txt
for wl in c2 c3; do timeout 200 python scripts/bench_module.py --workload $wl; done > gpurun_out/m1_bench.jsonl 2> gpurun_out/m1_bench.err
timeout 300 ncu --set full --import-source on --clock-control none -k regex:om_linear -c 2 -o /tmp/oml python scripts/bench_module.py --workload c2 --reps 1 > gpurun_out/m1_ncu.log 2>&1
ncu -i /tmp/oml.ncu-rep --page raw --csv > gpurun_out/m1_oml_raw.csv 2>&1
