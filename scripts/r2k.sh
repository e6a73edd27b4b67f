set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py -q -x > gpurun_out/r2l_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/r2l_pytest.txt
timeout 600 python scripts/tune.py --workload c4 --passes bwd --reps 10 > gpurun_out/r2l_tune_c4.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bwd33 -c 1 -o gpurun_out/r2l_bwd33_c4s1 python scripts/profile_stage.py --workload c4 --stage 0 --batch 128 --reps 1 > gpurun_out/r2l_ncu.log 2>&1
