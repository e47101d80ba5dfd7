# Bench the c2 s values under environment settings.  Usage: bash scripts/gpu/s_env.sh "S1 S2 ..." "A=1" ...
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SS=$1; shift
for s in $SS; do for e in "NONE=0" "$@"; do
env $e timeout 600 python bench.py --s $s --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/senv.json 2>&1
python - "gpurun_out/senv.json" "$e" "$s" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[2], open(sys.argv[1]).read()[-600:]); sys.exit()
d=json.loads(l[-1])
print(f"s={sys.argv[3]:5s} [{sys.argv[2]:20s}] value {d['value']:.1f} support {d['support_exact']}")
PY
done; done
