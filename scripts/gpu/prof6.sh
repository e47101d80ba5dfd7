cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain10.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k1_gather" -s 5 -c 1 -o gpurun_out/prof_r1h $CMD > gpurun_out/ncu_full10.log 2>&1 ; echo "full rc=$?"
