# quick iteration: GPU parity tests, then bench variants (env VARIANTS="SGM_SEG=12 SGM_LPT=1;...")
if [ -z "$SKIP_TESTS" ]; then
  python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
  cat gpurun_out/pytest_gpu.log
fi
IFS=';' read -ra VS <<< "${VARIANTS:-SGM_SEG=12}"
i=0
for V in "${VS[@]}"; do
  env $V python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e ${BARGS} > gpurun_out/bench_v$i.json 2> gpurun_out/bench_v$i.err
  python -c "
import json
d=json.load(open('gpurun_out/bench_v$i.json'))
print('[$V] value %.3g ms/step %.4f step_gbs %.0f'%(d['value'],d['ms_per_step'],d['roofline']['step_gbs']))
for k,v in d['kernels'].items(): print('  %-14s %.1f us %6.0f GB/s'%(k,1e3*v['ms_per_launch'],v.get('gbs',0)))
" || tail -5 gpurun_out/bench_v$i.err
  i=$((i+1))
done
