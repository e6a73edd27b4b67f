#!/bin/bash
# Export an ncu report to CSV on the GPU box (raw metrics + cuda/sass source view) and drop
# the binary report when it is large, so gpurun_out/ stays under the 64 MiB copy-back limit.
#   bash scripts/ncu_export.sh gpurun_out/name.ncu-rep [max_mib]
rep="$1"; max="${2:-20}"
[ -f "$rep" ] || exit 0
base="${rep%.ncu-rep}"
ncu -i "$rep" --page raw --csv > "${base}_raw.csv" 2>/dev/null
ncu -i "$rep" --page source --csv --print-source cuda,sass > "${base}_src.csv" 2>/dev/null
gzip -f "${base}_src.csv"
size=$(( $(stat -c %s "$rep") / 1048576 ))
if [ "$size" -gt "$max" ]; then rm -f "$rep"; echo "dropped $rep (${size} MiB)"; fi
