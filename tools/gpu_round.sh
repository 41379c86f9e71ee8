# One GPU session: parity tests, smoke, bench line, ncu launch list + full capture of K1/K2.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-cache > gpurun_out/launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k1_streams|k2_warp" -c 2 -o gpurun_out/prof_full python bench.py --profile --steps 1 --warmup 1 --no-cache > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench.json
timeout 600 python bench.py --workload config2 --no-e2e --no-cpu --no-cache > gpurun_out/bench_config2.json 2>/dev/null
tail -1 gpurun_out/bench_config2.json
