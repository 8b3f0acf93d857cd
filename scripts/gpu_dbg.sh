for D in 0 1 2 3; do for NP in 2 4 8; do
  SGM_PIPE_DBG=$D SGM_NP=$NP SGM_NP_UPD=$NP python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/dbg_$D_$NP.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/dbg_$D_$NP.json'))
print('dbg=$D np=$NP', ' '.join('%s=%.1fus'%(k,1e3*v['ms_per_launch']) for k,v in d['kernels'].items()))
"
done; done
