set -x
for off in u2 u8; do
  timeout 300 python scripts/tune.py --workload c4 --offsets $off --reps 10 --batch 128 > gpurun_out/r2g_c4_$off.jsonl 2>&1
  DCNV4_FWD_PATH=g DCNV4_BWD_PATH=g timeout 300 python scripts/tune.py --workload c4 --offsets $off --reps 10 --batch 128 > gpurun_out/r2g_c4_${off}_generic.jsonl 2>&1
  timeout 300 python scripts/tune.py --workload c2_f16 --offsets $off --reps 10 > gpurun_out/r2g_c2f16_$off.jsonl 2>&1
  DCNV4_FWD_PATH=g timeout 300 python scripts/tune.py --workload c2_f16 --offsets $off --reps 10 > gpurun_out/r2g_c2f16_${off}_generic.jsonl 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bwd33 -c 1 -o gpurun_out/r2g_bwd33_c4s1 python scripts/profile_stage.py --workload c4 --stage 0 --batch 128 --reps 1 > gpurun_out/r2g_ncu1.log 2>&1

