set -x
for wl in c2_f32 c2_f16; do
 for th in 1 2 4 8; do DCNV4_FWD33_TH=$th python scripts/tune.py --workload $wl --passes fwd --stages 1,2,3 --reps 50 | sed "s/^/{\"th\": $th, \"wl\": \"$wl\", \"x\": /; s/$/}/"; done
 DCNV4_FWD_PATH=g python scripts/tune.py --workload $wl --passes fwd --stages 1,2,3 --reps 50 | sed "s/^/{\"th\": \"g\", \"wl\": \"$wl\", \"x\": /; s/$/}/"
 DCNV4_NONPERSISTENT=1 python scripts/tune.py --workload $wl --passes fwd --stages 1,2,3 --reps 50 | sed "s/^/{\"th\": \"np\", \"wl\": \"$wl\", \"x\": /; s/$/}/"
done
