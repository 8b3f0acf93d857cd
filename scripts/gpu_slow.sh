# full-size parity tests (pytest -m "gpu and slow"); K selects a subset
mkdir -p gpurun_out
python paper_2302_04979_b200/build.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 3000 python -m pytest tests -m "gpu and slow" -q -k "${K:-not nothing}" --durations=0 2>&1 | tail -40 | tee gpurun_out/slow_${TAG:-x}.log
