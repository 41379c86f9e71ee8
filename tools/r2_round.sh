# Round-2 GPU session: parity, smoke, bench (ours + reference arm), decode-only launch list, ncu full of K1/K2w.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/lscpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k_scan|k_region|k_unpack|k_plan" --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-cache --no-gather > gpurun_out/launch_bench.log 2>&1
bash tools/ncu_full.sh prof_r02
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt; tail -c 2500 gpurun_out/bench.json; tail -c 600 gpurun_out/ref.json
