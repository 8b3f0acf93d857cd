# round-2 evidence refresh (TAG) followed by the full-size parity tests
TAG=${TAG:-r2d} bash scripts/gpu_full_r2.sh > gpurun_out/full_${TAG:-r2d}.log 2>&1
timeout 3000 python -m pytest tests -m "gpu and slow" -q --durations=0 2>&1 | tail -40 > gpurun_out/slow_${TAG:-r2d}.log
tail -5 gpurun_out/slow_${TAG:-r2d}.log; cat gpurun_out/pytest_gpu_${TAG:-r2d}.log
