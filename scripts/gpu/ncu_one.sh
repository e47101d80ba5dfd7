# ncu --set full of one kernel launch of the bench.  Usage: bash scripts/gpu/ncu_one.sh TAG KREGEX SKIP COUNT
TAG=$1; KR=$2; SK=${3:-5}; CN=${4:-1}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s $SK -c $CN -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1 ; echo "full rc=$?"
tail -2 gpurun_out/ncu_full_$TAG.log | cut -c1-300
