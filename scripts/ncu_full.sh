# one ncu --set full capture of the sweep kernels of one step (bench config), single GPU
ARGS=${ARGS:-"--steps 3 --warmup 3 --no-cpu --no-e2e"}
TAG=${TAG:-r1}
KREGEX=${KREGEX:-"regex:sweep"}
SKIP=${SKIP:-30}
COUNT=${COUNT:-6}
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k $KREGEX --launch-skip $SKIP --launch-count $COUNT \
    -o gpurun_out/full_$TAG -f python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/full_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/full_$TAG.ncu-rep --page source --csv > gpurun_out/full_${TAG}_source.csv 2>/dev/null
ncu -i gpurun_out/full_$TAG.ncu-rep --page details --csv > gpurun_out/full_${TAG}_details.csv 2>/dev/null
