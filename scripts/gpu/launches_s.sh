# ncu launch list of one bench step at sparsity s.  Usage: bash scripts/gpu/launches_s.sh TAG S
TAG=$1; S=$2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --s $S --steps 1 --warmup 2 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; echo "launch rc=$?"
python scripts/launch_summary.py gpurun_out/launches_$TAG.csv 25
