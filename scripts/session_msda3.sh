timeout 600 python -m pytest tests/test_gpu_msda.py -q > gpurun_out/ms3_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/ms3_pytest.txt
MSDA_SCHED=persist timeout 600 python -m pytest tests/test_gpu_msda.py -q > gpurun_out/ms3_pytest_persist.txt 2>&1; echo "exit $?" >> gpurun_out/ms3_pytest_persist.txt
for v in "MSDA_SCHED=flat" "MSDA_SCHED=persist" "MSDA_SCHED=persist MSDA_VEC=1"; do
  for d in f32 bf16; do
    echo "== $v $d"; env $v python scripts/bench_msda.py --dtype $d --no-verify | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['passes'])"
  done
done > gpurun_out/ms3_ab.txt 2>&1
timeout 600 env MSDA_SCHED=persist ncu --set full --import-source on --clock-control none -k regex:msda_ -c 2 -o /tmp/ms3 python scripts/bench_msda.py --steps 1 --warmup 1 --no-verify > gpurun_out/ms3_ncu.log 2>&1
ncu -i /tmp/ms3.ncu-rep --page raw --csv > gpurun_out/ms3_raw.csv 2>&1
