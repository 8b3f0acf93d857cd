# one ncu --set full capture of the 6 sweep kernels of one step (bench config), single GPU
set -x
ARGS=${ARGS:-"--steps 3 --warmup 3 --no-cpu --no-e2e"}
TAG=${TAG:-r1}
ncu --set full --clock-control none --import-source on -k regex:seg_ --launch-skip 30 --launch-count 6 \
    -o gpurun_out/full_$TAG -f python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/full_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/full_$TAG.ncu-rep --page details --csv > gpurun_out/full_${TAG}_details.csv 2>/dev/null
ls -la gpurun_out
