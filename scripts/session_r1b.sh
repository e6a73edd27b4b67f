# Re-entry GPU session: parity, bench lines, MSDA measurement + ncu.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/s1_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s1_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/s1_bench_c4.json 2> gpurun_out/s1_bench_c4.err
for d in f32 f16 bf16; do timeout 300 python scripts/bench_msda.py --dtype $d; done > gpurun_out/s1_msda.jsonl 2> gpurun_out/s1_msda.err
for k in fwd bwd; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:msda_${k} -c 1 -o /tmp/msda_${k} \
     python scripts/bench_msda.py --steps 1 --warmup 1 --no-verify > gpurun_out/s1_ncu_msda_$k.log 2>&1
  ncu -i /tmp/msda_${k}.ncu-rep --page raw --csv > gpurun_out/s1_msda_${k}_raw.csv 2>&1
  ncu -i /tmp/msda_${k}.ncu-rep --page source --csv --print-source sass > gpurun_out/s1_msda_${k}_sass.csv 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s1_msda_launches.csv \
    python scripts/bench_msda.py --steps 2 --warmup 1 --no-verify > /dev/null 2>&1
