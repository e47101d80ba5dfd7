cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
LA=paper_1706_02740_b200/libdsft_a.so
echo "== lib A"; DSFT_LIB=$LA timeout 600 python scripts/kern_times.py 67108864 1000 "A:seed=0"
echo "== lib B"; timeout 600 python scripts/kern_times.py 67108864 1000 "B:seed=0"
for r in 1 2; do
DSFT_LIB=$LA timeout 600 python scripts/ab.py 67108864 1000 "A:seed=0" --reps 30 --rounds 2
timeout 600 python scripts/ab.py 67108864 1000 "B:seed=0" --reps 30 --rounds 2
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
