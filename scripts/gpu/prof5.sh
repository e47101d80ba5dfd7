cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain8.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k2_prime|k3_ident" -s 10 -c 2 -o gpurun_out/prof_r1g $CMD > gpurun_out/ncu_full8.log 2>&1 ; echo "full rc=$?"
