# Bench a list of DSFT_ORDER permutations.  Usage: bash scripts/gpu/order_sweep.sh "0,1,2,3,4" "4,0,1,2,3" ...
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in 1 2; do for o in "$@"; do
DSFT_ORDER="$o" timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ord_$o.json 2>&1
python - "gpurun_out/ord_$o.json" "$o" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); print(f"[{sys.argv[2]}] value {d['value']:.1f} ms {d['ms_per_step']:.4f}")
PY
done; done
