python -m pytest tests/test_gpu_parity.py -q -x -k "general or curved or cfl or composed" 2>&1 | tail -3
python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c4" 2>&1 | tail -3
for V in "X=1" "SGM_HODGE_PENCIL=1"; do
  for C in c4 c3; do
    env $V python bench.py --config $C --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/hb_$C.json 2>gpurun_out/hb_$C.err
    python -c "
import json; d=json.load(open('gpurun_out/hb_$C.json')); print('[$V $C] %.3g ms/step %.4f'%(d['value'],d['ms_per_step']), {k:round(1e3*v['ms_per_launch'],1) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/hb_$C.err
  done
done
