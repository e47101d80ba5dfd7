# A/B of a K3 change (A: current sources, B: libdsft_old.so) + parity.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${1:-kmj}
timeout 900 python -m pytest tests -m gpu -q -x -k "candidates or deterministic or headline_config_full_size or end_to_end or band_budget or sharded" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
timeout 300 python scripts/kern_times.py 67108864 1000 "c2:seed=0" > gpurun_out/kt_${T}_A.txt 2>&1; head -7 gpurun_out/kt_${T}_A.txt
DSFT_LIB=paper_1706_02740_b200/libdsft_old.so timeout 300 python scripts/kern_times.py 67108864 1000 "c2:seed=0" > gpurun_out/kt_${T}_B.txt 2>&1; head -7 gpurun_out/kt_${T}_B.txt
bash scripts/gpu/ab.sh $T paper_1706_02740_b200/libdsft_old.so
bash scripts/gpu/ab.sh ${T}2 paper_1706_02740_b200/libdsft_old.so
