# interleaved A/B of two prebuilt product libraries (paper_2302_04979_b200/libsgm_a.so vs libsgm_b.so)
# on one box: for each rep and config, copy one in as libsgm.so and time bench.py; prints ms per step
# and per-class kernel times.  TESTK: GPU tests run once on library B first.
L=paper_2302_04979_b200
mkdir -p gpurun_out
use() { cp $L/libsgm_$1.so $L/libsgm.so; touch $L/libsgm.so; }
if [ -n "$TESTK" ]; then use b; timeout 900 python -m pytest tests -m gpu -x -q -k "$TESTK" 2>&1 | tail -3; fi
for rep in $(seq 1 ${REPS:-2}); do
  for C in ${CONFS:---config c4}; do
    for V in a b; do
      use $V
      timeout 300 python bench.py $C --steps ${STEPS:-20} --warmup 5 --no-cpu --no-e2e --no-variants 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
ks=' '.join('%s=%.1f'%(k,1e3*v['ms_per_launch']) for k,v in d['kernels'].items())
print('%-16s %s %.4f ms/step  %s'%('$C'.replace('--config ',''),'$V',d['ms_per_step'],ks))"
    done
  done
done
use b
