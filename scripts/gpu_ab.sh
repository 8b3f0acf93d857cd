# interleaved A/B on one box: for each config, alternate variants REPS times; prints ms/step
IFS=';' read -ra VS <<< "${VARIANTS:-SGM_X=0;SGM_X=1}"
IFS='|' read -ra CS <<< "${CONFIGS:---p 3 --n 128}"
for C in "${CS[@]}"; do
  for rep in $(seq 1 ${REPS:-3}); do
    for V in "${VS[@]}"; do
      env $V timeout 120 python bench.py --steps ${STEPS:-64} --warmup ${WARM:-16} --no-cpu --no-e2e --no-variants $C 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
print('%-22s %-28s %.4f'%('$C','$V',d['ms_per_step']))"
    done
  done
done
