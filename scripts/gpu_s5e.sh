# refresh of the general-Hodge parts of the round-2 evidence (TAG): parity tests, C4/C3 bench lines, ncu captures
TAG=${TAG:-r2e}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
rm -f gpurun_out/bench_hodge_$TAG.jsonl
for cfg in "--config c4" "--config c3"; do
  python bench.py --steps 20 --warmup 5 --no-e2e $cfg >> gpurun_out/bench_hodge_$TAG.jsonl 2>> gpurun_out/bench_hodge_$TAG.err
done
ARGS="--steps 3 --warmup 3 --no-cpu --no-e2e --no-variants"
for c in c3 c4; do
  ncu --set full --clock-control none -k "regex:hodge_brick|hodge_gather" --launch-skip 4 --launch-count 2 \
      -o gpurun_out/hodge_${c}_$TAG -f python bench.py --config $c $ARGS > gpurun_out/ncu_hodge_${c}_$TAG.log 2>&1
  ncu -i gpurun_out/hodge_${c}_$TAG.ncu-rep --page raw --csv > gpurun_out/hodge_${c}_${TAG}_raw.csv 2>/dev/null
  rm -f gpurun_out/hodge_${c}_$TAG.ncu-rep
done
cat gpurun_out/pytest_gpu_$TAG.log gpurun_out/smoke_$TAG.log
