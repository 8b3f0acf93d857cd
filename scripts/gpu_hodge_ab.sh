# general-Hodge brick kernel: parity of both modes, then an interleaved A/B of C3 / C4 steps
# (group mode = options 0, layer-synchronous = 0x40); prints ms per step and per-class kernel times
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-general_hodge or scheme1 or c3 or c4 or hodge}" 2>&1 | tail -${TAILN:-5}
for rep in $(seq 1 ${REPS:-2}); do
  for C in ${CONFS:-c4 c3}; do
    for O in 0 0x40; do
      timeout 300 python bench.py --config $C --steps ${STEPS:-20} --warmup 5 --no-cpu --no-e2e --no-variants --opts $O 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
ks=' '.join('%s=%.1f'%(k,1e3*v['ms_per_launch']) for k,v in d['kernels'].items())
print('%-4s opts=%-5s %.4f ms/step  %s'%('$C','$O',d['ms_per_step'],ks))"
    done
  done
done
