# brick-kernel iteration: Hodge parity tests, then the C3 / C4 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x -k "${KEXPR:-hodge or general or otf or scheme1 or mass or curved or coax or lift or pcg}" 2>&1 | tail -8
for c in c4 c3; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e ${VARIANTS:---no-variants} > gpurun_out/bench_${c}_${TAG:-s5b}.json 2> gpurun_out/bench_${c}_${TAG:-s5b}.err
  python - <<PY
import json
d=json.load(open('gpurun_out/bench_${c}_${TAG:-s5b}.json'))
print('$c ms/step %.4f'%d['ms_per_step'], 'value %.3e'%d['value'])
for k,v in d['kernels'].items(): print('   ', k, 'ms %.4f'%v['ms_per_launch'], 'x%d'%v['launches'])
PY
done
