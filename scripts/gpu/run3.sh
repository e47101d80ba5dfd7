cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not headline" > gpurun_out/pytest3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest3.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain6.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k1_gather|k4_vote|k5_est|k6_merge" -s 8 -c 8 -o gpurun_out/prof_r1e $CMD > gpurun_out/ncu_full5.log 2>&1 ; echo "full rc=$?"
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench3.log') if x.startswith('{')]
d=json.loads(l[-1]); print('value',d['value'],'ms',d['ms_per_step'],'support',d['support_exact']); print('roof',d['roofline']['achieved'],d['roofline']['frac'])
for k,v in d['kernels'].items(): print(k, v)
PY
