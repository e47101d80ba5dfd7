# Round-2 (session 4) evidence run on the final sources, without the all-configs sweep (scripts/configs.py runs in its own call).  Usage: bash scripts/gpu/final_r2f.sh TAG
TAG=${1:-r2c}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_1706_02740_b200.build > /dev/null || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
# ncu capture of K1/K2/K3 first, so the bench below reports measured traffic for these sources
python scripts/run_one.py 67108864 1000 2 flags=32 > gpurun_out/plain1_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k1_gather|k2_ct|k3_ident" -s 0 -c 15 -o gpurun_out/prof_$TAG python scripts/run_one.py 67108864 1000 2 flags=32 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full rc=$?"
python scripts/ncu_traffic.py gpurun_out/prof_$TAG.ncu-rep --capture "ncu --set full --clock-control none --import-source on -k regex:'k1_gather|k2_ct|k3_ident' -s 0 -c 15 python scripts/run_one.py 67108864 1000 2 flags=32 (BASELINE config 2, round-2 final sources, cold caches per kernel replay)"; echo "traffic rc=$?"
cp profiles/traffic.json gpurun_out/traffic_$TAG.json
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 600 python scripts/latency.py --out gpurun_out/latency_$TAG.json > gpurun_out/latency_$TAG.log 2>&1; echo "latency rc=$?"
timeout 600 python scripts/timeline.py 67108864 1000 > gpurun_out/timeline_$TAG.txt 2>&1
timeout 600 python scripts/kern_times.py 67108864 1000 "c2:seed=0" > gpurun_out/kern_times_$TAG.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch rc=$?"

