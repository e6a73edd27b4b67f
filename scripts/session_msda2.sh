timeout 600 python -m pytest tests/test_gpu_msda.py -q > gpurun_out/ms2_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/ms2_pytest.txt
for v in "MSDA_GRID_CAP=1 MSDA_VEC=0" "MSDA_GRID_CAP=1" "MSDA_VEC=0" ""; do
  for d in f32 bf16; do
    echo "== $v $d"; env $v python scripts/bench_msda.py --dtype $d --no-verify | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['passes'])"
  done
done > gpurun_out/ms2_ab.txt 2>&1
for d in f32 f16 bf16; do timeout 300 python scripts/bench_msda.py --dtype $d; done > gpurun_out/ms2_bench.jsonl 2> gpurun_out/ms2_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:msda_ -c 2 -o /tmp/ms2 python scripts/bench_msda.py --steps 1 --warmup 1 --no-verify > gpurun_out/ms2_ncu.log 2>&1
ncu -i /tmp/ms2.ncu-rep --page raw --csv > gpurun_out/ms2_raw.csv 2>&1
