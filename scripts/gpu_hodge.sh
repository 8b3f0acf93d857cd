python -m pytest tests/test_gpu_parity.py -q -x -k "general" 2>&1 | tail -2
python -m pytest tests/test_gpu_fullsize.py -q -x -k "c4 or c3" 2>&1 | tail -2
for V in ${HV:-"SGM_HODGE_PENCIL=1" "SGM_HODGE_PENCIL=0"}; do for c in c4 c3; do env $V python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e | python -c "
import json,sys; d=json.load(sys.stdin); print('$V', d['config']['workload'][:30], '%.3g'%d['value'], '%.3f ms'%d['ms_per_step'], 'hodge %.1f us'%(1e3*d['kernels']['hodge_general']['ms_per_launch']))"; done; done
