# session check: parity tests (not slow), default bench, ncu source-level capture of the C4 brick kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_s5a.log
python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_s5a.json 2> gpurun_out/bench_s5a.err
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-variants > gpurun_out/bench_c4_s5a.json 2> gpurun_out/bench_c4_s5a.err
TAG=c4src KREGEX=hodge_brick SKIP=4 SOURCE=1 ARGS="--config c4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-variants" bash scripts/ncu_one.sh
gzip -f gpurun_out/ncu_c4src_source.csv
cat gpurun_out/pytest_gpu_s5a.log
head -c 600 gpurun_out/bench_s5a.json; echo
head -c 400 gpurun_out/bench_c4_s5a.json
