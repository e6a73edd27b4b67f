set -x
timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_parity.py -q -x > gpurun_out/r2h_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/r2h_pytest.txt
for wl in c3_f16 c3_f16_grouped c2_f16 c2_f16_grouped; do for b in 1 8; do timeout 300 python bench.py --workload $wl --global-batch $b --no-cpu-baseline --warmup 5; done; done > gpurun_out/r2h_grouped.jsonl 2> gpurun_out/r2h_grouped.err
timeout 300 python bench.py --workload c2_f16_grouped --no-cpu-baseline --warmup 5 >> gpurun_out/r2h_grouped.jsonl 2>> gpurun_out/r2h_grouped.err
timeout 300 python bench.py --workload c2_f16 --no-cpu-baseline --warmup 5 >> gpurun_out/r2h_grouped.jsonl 2>> gpurun_out/r2h_grouped.err
