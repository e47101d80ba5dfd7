cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv $CMD > gpurun_out/ncu_launch3.log 2>&1 ; echo "launch rc=$?"
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k1_gather|k4_vote|k5_est|k6_merge" -s 20 -c 5 -o gpurun_out/prof_r1c $CMD > gpurun_out/ncu_full3.log 2>&1 ; echo "full rc=$?"
