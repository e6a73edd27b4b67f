timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/s2_pytest_gpu.txt
for wl in c4 c2_f16 c2_f32; do for off in u2 zero u8 smooth; do
  timeout 300 python bench.py --workload $wl --offsets $off --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1
done; done > gpurun_out/s2_sens.jsonl 2> gpurun_out/s2_sens.err
