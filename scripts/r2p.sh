set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py -q -x > gpurun_out/r2p_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/r2p_pytest.txt
timeout 600 python scripts/tune.py --workload c4 --passes bwd --reps 10 > gpurun_out/r2p_tune_c4.jsonl 2>&1
timeout 600 python scripts/tune.py --workload c5_bf16 --passes bwd --reps 10 > gpurun_out/r2p_tune_c5.jsonl 2>&1
