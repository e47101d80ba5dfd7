# Round check on one B200: smoke, GPU parity, bench (default args), launch list,
# ncu --set full of the top kernels.  Usage: bash scripts/gpu/full_check.sh TAG
TAG=${1:-x}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - "$TAG" <<'PY'
import json,sys
t=sys.argv[1]
l=[x for x in open(f'gpurun_out/bench_{t}.json') if x.startswith('{')]
if not l: print(open(f'gpurun_out/bench_{t}.err').read()[-3000:]); sys.exit()
d=json.loads(l[-1]); print('value',d['value'],'ms',d['ms_per_step'],'support',d['support_exact'],'clocks',d.get('clocks'))
print('roof',json.dumps(d['roofline'])[:400])
for k,v in d['kernels'].items(): print(k, v)
print('e2e', d['e2e']); print('cpu', d['cpu_baseline'])
PY
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k1_gather|k2_prime|k3_ident}" -s ${KSKIP:-20} -c ${KCOUNT:-3} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1 ; echo "full rc=$?"
tail -2 gpurun_out/ncu_full_$TAG.log | cut -c1-300
