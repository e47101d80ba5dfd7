# K2 warp-group experiment: serial per-launch K2 times and the pipelined step
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_1706_02740_b200.build > /dev/null || exit 1
V="base:seed=0"; for ws in 1 2 3; do for g in 1 2; do V="$V w${ws}g$g:seed=0,DSFT_X_K2_WS=$ws,DSFT_X_K2_G=$g"; done; done
timeout 900 python scripts/kern_times.py 67108864 1000 $V
timeout 600 python scripts/ab.py 67108864 1000 $V --reps 30 --rounds 2
