# Round-2 evidence run on one B200: parity tests (not slow), smoke, bench (default + reference arm),
# other workloads, configs[4] sweep, ncu launch list and full captures.  TAG names the files.
set -o pipefail
TAG=${TAG:-r2}
mkdir -p gpurun_out
python paper_2302_04979_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_$TAG.txt
timeout 1200 python -m pytest tests -m "gpu and not slow" -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
rm -f gpurun_out/bench_sweep_$TAG.jsonl
for cfg in "--p 2 --n 160" "--p 4 --n 128" "--p 3 --n 64" "--config c2" "--config c4" "--config c3"; do
  python bench.py --steps 20 --warmup 5 --no-e2e $cfg >> gpurun_out/bench_sweep_$TAG.jsonl 2>> gpurun_out/bench_sweep_$TAG.err
done
python scripts/c5_sweep.py --out gpurun_out/c5_sweep_$TAG.jsonl > gpurun_out/c5_sweep_$TAG.log 2>&1
ARGS="--steps 3 --warmup 3 --no-cpu --no-e2e --no-variants"
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:sweep_kernel|update_kernel" \
    --launch-skip ${SKIP:-26} --launch-count 14 -o gpurun_out/full_$TAG -f python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/full_${TAG}_raw.csv 2>/dev/null
rm -f gpurun_out/full_$TAG.ncu-rep
for c in c3 c4; do
  ncu --set full --clock-control none -k "regex:hodge_brick|hodge_gather" --launch-skip 4 --launch-count 2 \
      -o gpurun_out/hodge_${c}_$TAG -f python bench.py --config $c $ARGS > gpurun_out/ncu_hodge_${c}_$TAG.log 2>&1
  ncu -i gpurun_out/hodge_${c}_$TAG.ncu-rep --page raw --csv > gpurun_out/hodge_${c}_${TAG}_raw.csv 2>/dev/null
  rm -f gpurun_out/hodge_${c}_$TAG.ncu-rep
done
ls -la gpurun_out | tail -40
