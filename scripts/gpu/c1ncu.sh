cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_1706_02740_b200.build > /dev/null || exit 1
python scripts/run_one.py 4194304 50 3 > gpurun_out/c1plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size --clock-control none --cache-control none --csv --log-file gpurun_out/c1_launches.csv python scripts/run_one.py 4194304 50 3 > gpurun_out/c1ncu.log 2>&1
echo rc=$?
