set -x
for wl in module_full_c2 module_full_train_c2 module_c2; do timeout 600 python bench.py --workload $wl --warmup 5; done > gpurun_out/r2f_module_full.jsonl 2> gpurun_out/r2f_module_full.err
tail -5 gpurun_out/r2f_module_full.err
