for o in 0 1 0 1; do DCNV4_P4ORDER=$o python scripts/tune.py --workload c4 --passes bwd --reps 10 | sed "s/^/{\"ord\": $o, \"x\": /; s/$/}/"; done
for o in 0 1; do DCNV4_P4ORDER=$o python scripts/tune.py --workload c5_bf16 --passes bwd --reps 10 | sed "s/^/{\"ord\": $o, \"x\": /; s/$/}/"; done
