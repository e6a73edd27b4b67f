set -x
timeout 300 python -m pytest tests/test_gpu_module.py -q > gpurun_out/m3_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/m3_pytest.txt
for wl in c2 c3; do timeout 200 python scripts/bench_module.py --workload $wl; done > gpurun_out/m3_bench.jsonl 2> gpurun_out/m3_bench.err
timeout 300 ncu --set full --import-source on --clock-control none -k regex:module_fwd -c 1 -o /tmp/mf python scripts/bench_module.py --workload c2 --reps 1 > gpurun_out/m3_ncu.log 2>&1
ncu -i /tmp/mf.ncu-rep --page raw --csv > gpurun_out/m3_mf_raw.csv 2>&1
ncu -i /tmp/mf.ncu-rep --page source --csv --print-source sass > gpurun_out/m3_mf_sass.csv 2>&1
