# ncu launch list (per-kernel durations, serialised) of one bench step.  Usage: bash scripts/gpu/launches.sh TAG
TAG=$1
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; echo "launch rc=$?"
python scripts/launch_summary.py gpurun_out/launches_$TAG.csv
