cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
LA=paper_1706_02740_b200/libdsft_a.so
echo "== lib A (before the FMA DFT-3)"; DSFT_LIB=$LA timeout 600 python scripts/kern_times.py 67108864 1000 "base:seed=0" "pf:seed=0,DSFT_X_K2_PF=1"
echo "== lib B"; timeout 600 python scripts/kern_times.py 67108864 1000 "base:seed=0" "pf:seed=0,DSFT_X_K2_PF=1"
for r in 1 2; do
DSFT_LIB=$LA timeout 600 python scripts/ab.py 67108864 1000 "A:seed=0" "Apf:seed=0,DSFT_X_K2_PF=1" --reps 30 --rounds 2
timeout 600 python scripts/ab.py 67108864 1000 "B:seed=0" "Bpf:seed=0,DSFT_X_K2_PF=1" --reps 30 --rounds 2
done
