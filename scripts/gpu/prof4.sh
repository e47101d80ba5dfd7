cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain5.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k4_vote|k5_est|k6_merge" -s 3 -c 3 -o gpurun_out/prof_r1d $CMD > gpurun_out/ncu_full4.log 2>&1 ; echo "full rc=$?"
