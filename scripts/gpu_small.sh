python paper_2302_04979_b200/build.py > /dev/null 2>&1
for PN in "--config c2" "--p 3 --n 48" "--p 3 --n 64" "--p 2 --n 32" "--p 4 --n 32" "--p 3 --n 96"; do
  for O in 0 0x10; do
    python bench.py $PN --opts $O --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/s.json 2>gpurun_out/s.err && python -c "
import json; d=json.load(open('gpurun_out/s.json')); print('$PN', '$O', 'ms %.4f'%d['ms_per_step'], 'launches/step', d['schedule']['kernels_per_step'])" || tail -2 gpurun_out/s.err
  done
done
