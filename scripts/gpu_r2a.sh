# round-2 check: new GPU tests, fp64 peak, bench lines for C5 / C3 / C4
mkdir -p gpurun_out
python paper_2302_04979_b200/build.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -5
python scripts/fp64_peak.py r2 2>&1 | tail -1
for C in c5 c3 c4; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-e2e > gpurun_out/r2a_$C.json 2> gpurun_out/r2a_$C.err
  python -c "
import json; d=json.load(open('gpurun_out/r2a_$C.json')); r=d['roofline']
print('$C', 'ms %.4f'%d['ms_per_step'], 'val %.3e'%d['value'], 'dom', r['kernel'], 'frac', r['frac'], 'step_frac %.3f'%r['step_frac'], 'useful %.3f'%r['useful_bytes_frac'])
for k,v in r['functions'].items(): print('   ', k, {a:(round(b,4) if isinstance(b,float) else b) for a,b in v.items() if a!='classes'})
print('   variants', {k:(round(v['ms_per_step'],4), v['kernels_per_step']) for k,v in d['schedule_variants'].items()})
print('   cpu', d.get('cpu_baseline'))
" || tail -5 gpurun_out/r2a_$C.err
done
