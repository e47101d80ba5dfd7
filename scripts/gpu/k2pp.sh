cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_1706_02740_b200.build > /dev/null || exit 1
V="base:seed=0 pp512:seed=0,DSFT_X_K2_PP=512 pp384:seed=0,DSFT_X_K2_PP=384 pp768:seed=0,DSFT_X_K2_PP=768 pp256:seed=0,DSFT_X_K2_PP=256"
timeout 600 python scripts/kern_times.py 67108864 1000 $V
timeout 600 python scripts/ab.py 67108864 1000 $V --reps 30 --rounds 2
