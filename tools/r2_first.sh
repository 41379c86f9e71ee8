set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_streams|k2_warp|k_scan|k_region|k2_replay|k_unpack|k_plan" --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-cache > gpurun_out/launch_bench.log 2>&1
cat gpurun_out/pytest_gpu.txt; tail -c 3000 gpurun_out/bench.json
