# One ncu --set full capture of K1 + K2w on config 3 (bench.py --profile), report into gpurun_out/.
# usage: bash tools/ncu_full.sh NAME [extra bench args]
name=${1:-prof}; shift
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k1_streams|k1_fast|k2_warp" -c 2 \
  -o gpurun_out/$name python bench.py --profile --steps 1 --warmup 1 --no-cache "$@" > gpurun_out/$name.log 2>&1
tail -3 gpurun_out/$name.log
