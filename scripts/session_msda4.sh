timeout 600 python -m pytest tests/test_gpu_msda.py -q > gpurun_out/ms4_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/ms4_pytest.txt
for v in "MSDA_BWD8=0" "MSDA_BWD8=1"; do for d in f16 bf16; do
  echo "== $v $d"; env $v python scripts/bench_msda.py --dtype $d --no-verify | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['passes'])"
done; done > gpurun_out/ms4_ab.txt 2>&1
for d in f32 f16 bf16; do timeout 300 python scripts/bench_msda.py --dtype $d; done > gpurun_out/ms4_bench.jsonl 2> gpurun_out/ms4_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ms4_launches.csv python scripts/bench_msda.py --steps 2 --warmup 1 --no-verify > /dev/null 2>&1
