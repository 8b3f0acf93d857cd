# ncu source-level captures of the brick kernel (CFGS, default c4)
mkdir -p gpurun_out
for c in ${CFGS:-c4}; do
TAG=${c}src KREGEX=hodge_brick SKIP=4 SOURCE=1 ARGS="--config $c --steps 3 --warmup 3 --no-cpu --no-e2e --no-variants" bash scripts/ncu_one.sh
gzip -f gpurun_out/ncu_${c}src_source.csv
done
