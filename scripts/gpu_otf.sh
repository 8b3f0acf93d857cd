mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "otf or rational or general_hodge" 2>&1 | tail -15
for r in 1 2; do
timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
print('c3 %.4f ms/step'%d['ms_per_step'], json.dumps(d['schedule_variants']), 'hodge', d['kernels']['hodge_general']['ms_per_launch'])"
done
