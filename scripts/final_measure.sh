# Round-end measurement bundle (one gpurun call): bench lines, launch list, ncu summaries,
# traffic, sanitizers.  Outputs land in gpurun_out/final_*.
set -x
python bench.py > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.err
for wl in c2_f32 c2_f16 c3_f16 c5_bf16; do python bench.py --workload $wl --steps 30 --warmup 5; done > gpurun_out/final_sweep.jsonl 2> gpurun_out/final_sweep.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-verify --e2e-steps 1 > gpurun_out/final_ncu_bench.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/final_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-verify --e2e-steps 1 > gpurun_out/final_ncu_traffic.log 2>&1
for k in fwd bwd; do
  extra=""; [ $k = fwd ] && extra="--fwd-only"
  ncu --set full --import-source on --clock-control none -k regex:${k}33 -c 1 -o /tmp/final_${k}_s1 \
      python scripts/profile_stage.py --workload c4 --stage 0 --batch 128 --reps 1 $extra > gpurun_out/final_ncu_$k.log 2>&1
  ncu -i /tmp/final_${k}_s1.ncu-rep --page raw --csv > gpurun_out/final_${k}_raw.csv 2>&1
  ncu -i /tmp/final_${k}_s1.ncu-rep --page source --csv --print-source sass > gpurun_out/final_${k}_sass.csv 2>&1
done
python scripts/bench_msda.py > gpurun_out/final_msda_f32.json 2> gpurun_out/final_msda.err
python scripts/bench_msda.py --dtype bf16 > gpurun_out/final_msda_bf16.json 2>> gpurun_out/final_msda.err
for t in memcheck racecheck synccheck initcheck; do echo "== compute-sanitizer --tool $t python scripts/sanitize_case.py"; \
  compute-sanitizer --tool $t python scripts/sanitize_case.py 2>&1 | grep -v "^=========  " | tail -8; done > gpurun_out/final_sanitizer.txt 2>&1
