# Bench a list of environment settings (e.g. "DSFT_K1GROUPS=1,4").  Usage: bash scripts/gpu/env_sweep.sh "A=1" "B=2" ...
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in 1 2; do for e in "NONE=0" "$@"; do
env $e timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/envsw.json 2>&1
python - "gpurun_out/envsw.json" "$e" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-800:]); sys.exit()
d=json.loads(l[-1]); k=d['kernels']
print(f"[{sys.argv[2]:22s}] value {d['value']:.1f} ms {d['ms_per_step']:.4f} support {d['support_exact']} k1 {k['k1_gather_mix']['ms_per_step']*1e3:.0f} k2 {k['k2_prime_dft']['ms_per_step']*1e3:.0f} k3 {k['k3_identify_vote']['ms_per_step']*1e3:.0f}")
PY
done; done
