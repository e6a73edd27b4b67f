# Measurement bundle (run under gpurun from the repo root): tests, smoke, sanitizer on the new kernels, bench lines,
# reference arm, launch list, ncu of the dominant kernel, CPU baseline protocol.
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/b_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/b_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.txt 2>&1; echo "exit $?" >> gpurun_out/b_smoke.txt
timeout 900 python bench.py > gpurun_out/b_bench_c4.json 2> gpurun_out/b_bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
for wl in module_full_c2 module_full_train_c2 module_c2 module_c3 c5_bf16; do timeout 300 python bench.py --workload $wl --warmup 5 --no-cpu-baseline; done > gpurun_out/b_workloads.jsonl 2> gpurun_out/b_workloads.err
for d in f32 f16 bf16; do timeout 300 python scripts/bench_msda.py --dtype $d; done > gpurun_out/b_msda.jsonl 2> gpurun_out/b_msda.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-verify --e2e-steps 1 --no-extras > gpurun_out/b_ncu_bench.log 2>&1
timeout 900 python scripts/cpu_baseline.py --out gpurun_out/b_cpu_baseline.json > gpurun_out/b_cpu_baseline.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/b_traffic_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-verify --e2e-steps 1 --no-extras > gpurun_out/b_traffic.log 2>&1
for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_r2.py > gpurun_out/b_sanitize_$tool.txt 2>&1; done
