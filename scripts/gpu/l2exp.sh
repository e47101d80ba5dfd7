cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for G in 0 32 64 128; do
  if [ "$G" = "0" ]; then unset DSFT_L2_FETCH; else export DSFT_L2_FETCH=$G; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/l2_$G.log 2>&1
  python - "$G" <<'PY'
import json,sys
l=[x for x in open(f'gpurun_out/l2_{sys.argv[1]}.log') if x.startswith('{')]
d=json.loads(l[-1]); print('G',sys.argv[1],'value',round(d['value'],1),'k1 ms',round(d['kernels']['k1_gather_mix']['ms_per_step'],4),'k2',round(d['kernels']['k2_prime_dft']['ms_per_step'],4),'frac',round(d['roofline']['frac'],3))
PY
done
export DSFT_L2_FETCH=32
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain9.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --cache-control none -k regex:k1_gather -c 5 --csv --log-file gpurun_out/k1_l2_32.csv $CMD > /dev/null 2>&1; echo ncu rc=$?
