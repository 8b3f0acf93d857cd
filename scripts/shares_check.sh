for A in "--p 2 --n 128" "--p 2 --n 160" "--p 3 --n 128" "--p 3 --n 160" "--p 4 --n 128" "--p 4 --n 160"; do
  for V in X=1; do
    env $V python bench.py $A --steps 30 --warmup 5 --no-cpu --no-e2e | python -c "import json,sys; d=json.load(sys.stdin); print('$A', round(1e3*d['ms_per_step'],1), {k:round(1e3*v['ms_per_launch'],1) for k,v in d['kernels'].items()})"
  done
done
