# Round-2 GPU check: smoke, GPU parity suite, bench (single + sharded modes at N=1).
# Usage: bash scripts/gpu/r2_check.sh TAG [pytest -k expr]
TAG=${1:-x}; KEXPR=${2:-}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,memory.free --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
if [ -n "$KEXPR" ]; then timeout 2400 python -m pytest tests -m gpu -q -k "$KEXPR" > gpurun_out/pytest_$TAG.log 2>&1; else timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; fi
echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_$TAG.log | tail -15 | cut -c1-300
for MODE in single batched-sharded band-sharded; do
  timeout 600 python bench.py --steps 30 --warmup 3 --mode $MODE --no-cpu-baseline $( [ $MODE != single ] && echo --no-e2e ) > gpurun_out/bench_${TAG}_$MODE.json 2> gpurun_out/bench_${TAG}_$MODE.err; echo "bench $MODE rc=$?"
done
python - "$TAG" <<'PY'
import json,sys
t=sys.argv[1]
for m in ("single","batched-sharded","band-sharded"):
    try:
        l=[x for x in open(f'gpurun_out/bench_{t}_{m}.json') if x.startswith('{')]
    except Exception as e:
        print(m, e); continue
    if not l: print(m, open(f'gpurun_out/bench_{t}_{m}.err').read()[-2000:]); continue
    d=json.loads(l[-1]); print(m,'value',round(d['value'],1),'ms',round(d['ms_per_step'],4),'support',d['support_exact'],'clocks',d.get('clocks'))
    print('  roof K2', round(d['roofline']['frac'],4), 'busy', d['roofline']['busy']['frac'], ' K1', round(d['roofline_gather']['frac'],4))
    for k,v in d['kernels'].items(): print(f"  {k:20s} {v['ms_per_step']*1e3:8.1f} us busy {v['busy_ms_per_step']*1e3:8.1f} x{v['launches_per_step']:.0f}")
    if d.get('e2e'): print('  e2e', {k: d['e2e'][k] for k in ('value','mode','h2d_bytes_per_step')})
PY
