# ncu --set full of one kernel class on a short run (after the same command ran clean).
# Usage: bash scripts/gpu/ncu_kernel.sh TAG REGEX SKIP COUNT N s [key=value ...]
# NCU_EXTRA (env): extra ncu options, e.g. "--cache-control none" for a warm-L2 capture
TAG=$1; RE=$2; SKIP=$3; CNT=$4; shift 4
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python scripts/run_one.py $1 $2 2 flags=32 ${@:3}"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none $NCU_EXTRA --import-source on -k regex:"$RE" -s $SKIP -c $CNT -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$TAG.log | cut -c1-300
