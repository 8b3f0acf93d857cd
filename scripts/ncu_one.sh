# ncu --set full of one launch of kernel KREGEX in `python bench.py $ARGS` (single GPU); the raw
# page (and the source page if SOURCE=1) is exported and the report itself left on the box
TAG=${TAG:-one}
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" --launch-skip ${SKIP:-2} --launch-count 1 \
    -o gpurun_out/ncu_$TAG -f python bench.py $ARGS > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${TAG}_raw.csv 2>/dev/null
if [ -n "$SOURCE" ]; then
  ncu -i gpurun_out/ncu_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_${TAG}_source.csv 2>/dev/null
fi
rm -f gpurun_out/ncu_$TAG.ncu-rep
tail -3 gpurun_out/ncu_$TAG.log
