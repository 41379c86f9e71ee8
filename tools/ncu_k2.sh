# ncu --set full of K2w alone (config 3), report into gpurun_out/NAME.ncu-rep
name=${1:-k2}; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_warp" -c 1 \
  -o gpurun_out/$name python bench.py --profile --steps 1 --warmup 1 --no-cache "$@" > gpurun_out/$name.log 2>&1
tail -2 gpurun_out/$name.log
