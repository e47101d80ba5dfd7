cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "not headline" > gpurun_out/pytest2.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest2.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench2.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print('value',d['value'],'ms',d['ms_per_step'],'support',d['support_exact']); print('roof',d['roofline']['achieved'],d['roofline']['frac'])
    for k,v in d['kernels'].items(): print(k, v)
    print('e2e', d['e2e'])
else:
    print(open('gpurun_out/bench2.log').read()[-3000:])
PY
