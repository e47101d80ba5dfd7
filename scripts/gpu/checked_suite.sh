# The GPU parity suite against the DSFT_CHECKED build (device bounds checks that trap,
# poisoned workspace + guard zones checked after every execute): this pool does not
# allow compute-sanitizer, so this is the memory-safety run.  Usage: bash scripts/gpu/checked_suite.sh TAG
TAG=${1:-chk}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_1706_02740_b200.build --checked > gpurun_out/build_checked_$TAG.log 2>&1 || { echo "checked build failed"; tail -5 gpurun_out/build_checked_$TAG.log; exit 1; }
export DSFT_LIB=$GRAFT_REPO_ROOT/paper_1706_02740_b200/libdsft_checked.so
export DSFT_JIT_CACHE=/tmp/dsft_jit_checked
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_checked_$TAG.log 2>&1; echo "checked pytest rc=$?"
grep -E "passed|failed|dsft check failed|guard zone" gpurun_out/pytest_checked_$TAG.log | tail -8 | cut -c1-300
