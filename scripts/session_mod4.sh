timeout 300 python -m pytest tests/test_gpu_module.py -q > gpurun_out/m4_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/m4_pytest.txt
for wl in c2 c3; do timeout 200 python scripts/bench_module.py --workload $wl; done > gpurun_out/m4_bench.jsonl 2> gpurun_out/m4_bench.err
for ps in 2 3 4; do DCNV4_MODULE_PER_SM=$ps python scripts/bench_module.py --workload c2 --reps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($ps, [r['fused_us'] for r in d['stages']])"; done > gpurun_out/m4_persm.txt 2>&1
