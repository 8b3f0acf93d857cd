# tuning-build variants: VARIANTS="ENV=..;ENV=.." CONFIGS="--p 3 --n 128|--p 2 --n 160" -> ms per step
IFS=';' read -ra VS <<< "${VARIANTS:-SGM_XWM=1000}"
IFS='|' read -ra CS <<< "${CONFIGS:---p 3 --n 128}"
for C in "${CS[@]}"; do
  for V in "${VS[@]}"; do
    for rep in ${REPS:-1}; do
      env $V timeout 120 python bench.py --steps ${STEPS:-30} --warmup ${WARM:-5} --no-cpu --no-e2e --no-variants $C 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
ks=' '.join('%s=%.1f'%(k,1e3*v['ms_per_launch']) for k,v in d['kernels'].items())
print('%-22s %-28s %.4f ms  %s'%('$C','$V',d['ms_per_step'],ks))"
    done
  done
done
