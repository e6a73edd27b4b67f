timeout 600 python -m pytest tests/test_gpu_msda.py -q 2>&1 | tail -1
for v in "MSDA_SHARE=0" "MSDA_SHARE=1"; do for d in f32 f16 bf16; do
  echo "== $v $d"; env $v python scripts/bench_msda.py --dtype $d --no-verify | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['passes']['fwd']['us'], d['passes']['bwd']['us'])"
done; done
