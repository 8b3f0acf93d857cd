# final refresh: general-Hodge evidence (TAG) and the full-size C3 / C4 parity tests on the final library
TAG=${TAG:-r2g} bash scripts/gpu_s5e.sh > gpurun_out/s5e_${TAG:-r2g}.log 2>&1
timeout 3000 python -m pytest tests -m "gpu and slow" -q --durations=0 2>&1 | tail -30 > gpurun_out/slow_${TAG:-r2g}.log
tail -4 gpurun_out/slow_${TAG:-r2g}.log; cat gpurun_out/pytest_gpu_${TAG:-r2g}.log
