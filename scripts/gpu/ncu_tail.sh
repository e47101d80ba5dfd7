# ncu of the tail kernels (K5b, K6) with dense warp-state sampling.  Usage: bash scripts/gpu/ncu_tail.sh TAG
TAG=${1:-tail}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --clock-control none \
  --import-source on -k regex:"k5b_select|k6_merge" -s 6 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$TAG.log | cut -c1-200
