for wl in c2_f32 c2_f16 c3_f16; do
 for th in 2 3 4 5 6 7 8; do DCNV4_FWD33_TH=$th python scripts/tune.py --workload $wl --passes fwd --reps 30 | sed "s/^/{\"th\": $th, \"wl\": \"$wl\", \"x\": /; s/$/}/"; done
done
for th in 2 4 5 6 7 8; do DCNV4_BWD33_TH=$th python scripts/tune.py --workload c2_f32 --batch 64 --passes bwd --reps 10 2>/dev/null | sed "s/^/{\"bth\": $th, \"wl\": \"c2bwd\", \"x\": /; s/$/}/"; done
