# K2 CTA-size experiment: serial per-launch K2 times and the pipelined step
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_1706_02740_b200.build > /dev/null || exit 1
V=""; for nt in 256 288 320 352 384; do V="$V n$nt:seed=0,DSFT_X_K2_NT=$nt,DSFT_X_K2_MINB=2"; done
timeout 600 python scripts/kern_times.py 67108864 1000 $V
timeout 600 python scripts/ab.py 67108864 1000 $V --reps 30 --rounds 3
