set -x
timeout 600 python scripts/tune.py --workload c4 --passes fwd --reps 10 > gpurun_out/r2m_tune_c4.jsonl 2>&1
timeout 600 python scripts/tune.py --workload c2_f16 --passes fwd --reps 10 > gpurun_out/r2m_tune_c2f16.jsonl 2>&1
timeout 600 python scripts/tune.py --workload c5_bf16 --reps 10 > gpurun_out/r2m_tune_c5.jsonl 2>&1
