set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
python bench.py --steps 20 --warmup 5 --p 2 --n 160 --no-cpu --no-e2e > gpurun_out/bench_p2.json 2>&1
python bench.py --steps 20 --warmup 5 --p 4 --n 128 --no-cpu --no-e2e > gpurun_out/bench_p4.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
