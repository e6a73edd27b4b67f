set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/r2a_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/r2a_bench_c4.json 2> gpurun_out/r2a_bench_c4.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bwd33 -c 1 -o gpurun_out/r2a_bwd33_c4s1 python scripts/profile_stage.py --workload c4 --stage 0 --batch 128 --reps 1 > gpurun_out/r2a_ncu_bwd.log 2>&1
tail -3 gpurun_out/r2a_ncu_bwd.log
