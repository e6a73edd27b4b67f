python scripts/sanitize_case.py > gpurun_out/san_plain.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do echo "== compute-sanitizer --tool $t python scripts/sanitize_case.py"; \
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize_case.py 2>&1 | grep -v "^=========  " | tail -14; done > gpurun_out/san.txt 2>&1
