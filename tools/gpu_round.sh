set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_streams|k2_fast" -c 2 -o gpurun_out/prof_full python bench.py --profile --steps 1 --warmup 1 --zlayers 16 --no-cache > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench.json
