cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ; echo "launch rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_gather|k2_prime|k3_ident|k45|k6_merge" -s 17 -c 5 -o gpurun_out/prof_r1a $CMD > gpurun_out/ncu_full.log 2>&1 ; echo "full rc=$?"
tail -5 gpurun_out/ncu_full.log
