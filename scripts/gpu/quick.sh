# Quick GPU iteration: parity tests + short bench summary.  Usage: bash scripts/gpu/quick.sh TAG [pytest -k expr]
TAG=${1:-q}; KEXPR=${2:-}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
if [ -n "$KEXPR" ]; then timeout 1200 python -m pytest tests -m gpu -q -x -k "$KEXPR" > gpurun_out/pytest_$TAG.log 2>&1; else timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; fi
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log | cut -c1-400
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - "$TAG" <<'PY'
import json,sys
t=sys.argv[1]
l=[x for x in open(f'gpurun_out/bench_{t}.json') if x.startswith('{')]
if not l: print(open(f'gpurun_out/bench_{t}.err').read()[-3000:]); sys.exit()
d=json.loads(l[-1]); print('value',round(d['value'],1),'ms',round(d['ms_per_step'],4),'support',d['support_exact'],'clocks',d.get('clocks'))
for k,v in d['kernels'].items(): print(f"  {k:20s} {v['ms_per_step']*1e3:8.1f} us  x{v['launches_per_step']:.0f}  {100*v['share']:.1f}%")
PY
