# A/B/C/D of JIT option sets.  Usage: bash scripts/gpu/ab3.sh TAG "opts1" "opts2" ...
TAG=$1; shift
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
i=0
for rep in 1 2; do for o in "" "$@"; do i=$((i+1))
DSFT_JIT_OPTS="$o" timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab3_${TAG}_$i.json 2>&1
python - "gpurun_out/ab3_${TAG}_$i.json" "$o" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); print(f"[{sys.argv[2]:30s}] value {d['value']:.1f} ms {d['ms_per_step']:.4f} k2 {d['kernels']['k2_prime_dft']['ms_per_step']*1e3:.1f}")
PY
done; done
