for th in 4 6 8; do DCNV4_BWD33_TH=$th python scripts/tune.py --workload c4 --passes bwd --reps 5 | sed "s/^/{\"bth\": $th, \"x\": /; s/$/}/"; done
