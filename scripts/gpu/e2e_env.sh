# e2e (dsft_execute_host) under environment settings.  Usage: bash scripts/gpu/e2e_env.sh "A=1" ...
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for e in "NONE=0" "$@"; do
env $e timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 10 > gpurun_out/e2eenv.json 2>&1
python - "gpurun_out/e2eenv.json" "$e" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-800:]); sys.exit()
d=json.loads(l[-1]); e=d['e2e']
print(f"[{sys.argv[2]:22s}] e2e {e['value']:.1f} ms {e['ms_per_step']:.3f} copy {e.get('copy_mode',{}).get('value')}")
PY
done
