# K2 CTA-shape experiment (plan-time knob DSFT_X_K2_NT / DSFT_X_K2_MINB)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_1706_02740_b200.build > /dev/null || exit 1
timeout 900 python scripts/ab.py 67108864 1000 "base:seed=0" "n128m3:seed=0,DSFT_X_K2_NT=128,DSFT_X_K2_MINB=3" \
  "n160m3:seed=0,DSFT_X_K2_NT=160,DSFT_X_K2_MINB=3" "n192m3:seed=0,DSFT_X_K2_NT=192,DSFT_X_K2_MINB=3" \
  "n96m3:seed=0,DSFT_X_K2_NT=96,DSFT_X_K2_MINB=3" "n128m2:seed=0,DSFT_X_K2_NT=128,DSFT_X_K2_MINB=2" --reps 30 --rounds 3
