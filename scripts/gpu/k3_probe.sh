# K3 in isolation vs in the pipeline: serial-schedule timeline, and ncu of the last
# K3 of one execute with caches kept warm.  Usage: bash scripts/gpu/k3_probe.sh
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
DSFT_SERIAL=1 python scripts/timeline.py 2>/dev/null | tail -18
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k3_ident" -s 19 -c 5 -o gpurun_out/prof_k3warm $CMD > gpurun_out/ncu_k3warm.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_k3warm.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,lts__t_sector_hit_rate.pct,dram__bytes_read.sum 2>/dev/null | cut -c1-400 | tail -6
