cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not headline" > gpurun_out/pytest4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest4.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench4.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench4.log').read()[-2000:])
d=json.loads(l[-1]); print('value',d['value'],'ms',d['ms_per_step'],'support',d['support_exact']); print('roof',d['roofline']['achieved'],d['roofline']['frac'])
for k,v in d['kernels'].items(): print(k, v)
PY
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain7.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv $CMD > gpurun_out/ncu_launch7.log 2>&1 ; echo "launch rc=$?"
