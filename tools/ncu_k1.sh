name=${1:-k1}; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_" -c 1 \
  -o gpurun_out/$name python bench.py --profile --steps 1 --warmup 1 --no-cache "$@" > gpurun_out/$name.log 2>&1
tail -2 gpurun_out/$name.log
