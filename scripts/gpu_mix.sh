mkdir -p gpurun_out
python paper_2302_04979_b200/build.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -4
show() { python -c "
import json,sys; d=json.load(open('$1')); r=d['roofline']
print('$2', 'ms %.4f'%d['ms_per_step'], 'val %.3e'%d['value'], 'sweep frac %.3f'%r['functions']['sweep']['frac'], 'step_frac %.3f'%r['step_frac'], {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items()})"; }
SGM_BUILD_TUNING=1 python paper_2302_04979_b200/build.py > gpurun_out/build_t.log 2>&1 || { tail -30 gpurun_out/build_t.log; exit 1; }
for PN in "--p 3 --n 128" "--p 2 --n 128" "--p 4 --n 128" "--p 3 --n 64" "--config c2" "--p 3 --n 160" "--p 2 --n 160"; do
  for V in "SGM_MIX=0" "SGM_MIX=1"; do
    env $V python bench.py $PN --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/l1.json 2>gpurun_out/l1.err && show gpurun_out/l1.json "$PN $V" || tail -3 gpurun_out/l1.err
  done
done
python paper_2302_04979_b200/build.py > /dev/null 2>&1
