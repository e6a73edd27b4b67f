ncu --set full --import-source on --clock-control none -k regex:bwd33 -c 1 -o gpurun_out/bwd_r1f_s1 python scripts/profile_stage.py --workload c4 --stage 0 --batch 128 --reps 1 > gpurun_out/ncu_bwd_r1f.log 2>&1
tail -3 gpurun_out/ncu_bwd_r1f.log
