timeout 600 python -m pytest tests/test_gpu_msda.py -q > gpurun_out/ms6_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/ms6_pytest.txt
for v in "MSDA_ORDER=m" "MSDA_ORDER=q"; do for d in f32 bf16; do
  echo "== $v $d"; env $v python scripts/bench_msda.py --dtype $d --no-verify | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['passes']['fwd']['us'], d['passes']['bwd']['us'])"
done; done > gpurun_out/ms6_ab.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:msda_ -c 2 -o /tmp/ms6 python scripts/bench_msda.py --steps 1 --warmup 1 --no-verify > gpurun_out/ms6_ncu.log 2>&1
ncu -i /tmp/ms6.ncu-rep --page raw --csv > gpurun_out/ms6_raw.csv 2>&1
