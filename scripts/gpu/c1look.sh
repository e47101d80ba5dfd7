cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_1706_02740_b200.build > /dev/null || exit 1
timeout 300 python scripts/latency.py --only c0,c1,c3,c2_s50 --reps 50 --out gpurun_out/lat_c1look.json 2>&1 | tail -8
timeout 300 python scripts/timeline.py 4194304 50 32
timeout 300 python scripts/kern_times.py 4194304 50 "c1:seed=0"
timeout 300 python scripts/run_one.py 4194304 50 2
