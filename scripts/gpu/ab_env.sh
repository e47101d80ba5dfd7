# A/B bench: default vs an environment setting.  Usage: bash scripts/gpu/ab_env.sh TAG "VAR=value" [bench args]
TAG=$1; ENVB=$2; shift 2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(open(sys.argv[1].replace('.json','.err')).read()[-2000:]); sys.exit()
d=json.loads(l[-1]); print('  value',round(d['value'],1),'ms',round(d['ms_per_step'],4),'support',d['support_exact'])
for k,v in d['kernels'].items(): print(f"    {k:20s} {v['ms_per_step']*1e3:8.1f} us  x{v['launches_per_step']:.0f}")
PY
}
for rep in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/abe_${TAG}_A$rep.json 2> gpurun_out/abe_${TAG}_A$rep.err; echo "A$rep (default)"; summ gpurun_out/abe_${TAG}_A$rep.json
env $ENVB timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/abe_${TAG}_B$rep.json 2> gpurun_out/abe_${TAG}_B$rep.err; echo "B$rep ($ENVB)"; summ gpurun_out/abe_${TAG}_B$rep.json
done
