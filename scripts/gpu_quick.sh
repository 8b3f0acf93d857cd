# quick GPU iteration: build, parity tests (not slow), bench of the default and unfused schedules
set -x
mkdir -p gpurun_out
python paper_2302_04979_b200/build.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q ${PYTEST_ARGS} 2>&1 | tail -25
for O in ${OPTS:-0 0x10}; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --opts $O ${BENCH_ARGS} > gpurun_out/bench_$O.json 2> gpurun_out/bench_$O.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/bench_$O.json'))
print('opts $O', d['config']['workload'], 'ms/step %.4f'%d['ms_per_step'], 'value %.3e'%d['value'], 'launches', d['gpu_launches'])
for k,v in d['kernels'].items(): print('   ', k, 'ms %.4f'%v['ms_per_launch'], 'x%d'%v['launches'], 'GB/s %s'%(round(v.get('gbs',0))))
" || tail -5 gpurun_out/bench_$O.err
done
