# Round-1 final bundle (re-entry session): tests, smoke, bench lines, reference arm, launch list.
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/f_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1; echo "exit $?" >> gpurun_out/f_smoke.txt
timeout 600 python bench.py > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
for wl in c2_f32 c2_f16 c3_f16 c5_bf16; do timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline; done > gpurun_out/f_sweep.jsonl 2> gpurun_out/f_sweep.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-verify --e2e-steps 1 > gpurun_out/f_ncu_bench.log 2>&1
for wl in c2 c3; do timeout 200 python scripts/bench_module.py --workload $wl; done > gpurun_out/f_module.jsonl 2> gpurun_out/f_module.err
for d in f32 f16 bf16; do timeout 300 python scripts/bench_msda.py --dtype $d; done > gpurun_out/f_msda.jsonl 2> gpurun_out/f_msda.err
