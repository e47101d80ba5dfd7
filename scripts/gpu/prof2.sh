cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k2_prime|k4_vote|k5_est|k6_merge|k3_ident|k1_gather" -s 18 -c 8 -o gpurun_out/prof_r1b $CMD > gpurun_out/ncu_full2.log 2>&1 ; echo "full rc=$?"
tail -3 gpurun_out/ncu_full2.log | cut -c1-300
