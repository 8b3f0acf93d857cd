# Full evidence run on one B200: parity tests, smoke, bench (default + reference arm), ncu launch
# list of the bench command, and one ncu --set full capture of one step's kernels.
set -o pipefail
TAG=${TAG:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_$TAG.txt
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
for cfg in "--p 2 --n 160" "--p 4 --n 128" "--p 3 --n 64" "--config c2" "--config c4" "--config c3"; do
  python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e $cfg >> gpurun_out/bench_sweep_$TAG.jsonl 2>> gpurun_out/bench_sweep_$TAG.err
done
python scripts/c5_sweep.py --out gpurun_out/c5_sweep_$TAG.jsonl > gpurun_out/c5_sweep_$TAG.log 2>&1
ARGS="--steps 3 --warmup 3 --no-cpu --no-e2e"
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
# one step = update, z, y, x (eps) + update, zy, x (mu); skip setup + warm-up launches, capture
# two steps (scripts/ncu_traffic.py picks one step starting at an Ampere update)
ncu --set full --clock-control none --import-source on -k "regex:sweep_kernel|update_kernel" \
    --launch-skip ${SKIP:-26} --launch-count 14 -o gpurun_out/full_$TAG -f python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/full_${TAG}_raw.csv 2>/dev/null
# keep the merge-back under 64 MiB: the report itself stays on the box
rm -f gpurun_out/full_$TAG.ncu-rep
ls -la gpurun_out | tail -30
