# compute-sanitizer over small transforms (one tool per call): BASELINE config 0
# (N = 4096, s = 8), a prime length N = 97, the small-plan path, the pipelined path
# (DSFT_FLAG_SERIAL and the four-stream default at N = 2^20, s = 2000: cluster K2),
# a general-prime pool, and the generic-kappa K1 (THM4).
# Usage: bash scripts/gpu/sanitize.sh TOOL   (memcheck | racecheck | synccheck | initcheck)
TOOL=${1:-memcheck}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
OUT=gpurun_out/sanitize_$TOOL.txt
: > $OUT
run() {
  echo "=== $*" >> $OUT
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 20 python scripts/run_one.py "$@" >> $OUT 2>&1
  echo "rc=$?" >> $OUT
}
run 4096 8 2
run 97 4 2
run 4194304 50 2
run 1048576 2000 1 flags=16
run 1048576 2000 1
run 65536 50 1 pool_rule=full
run 65536 20 1 preset=thm4 r=2
grep -E "^===|rc=|ERROR SUMMARY" $OUT
