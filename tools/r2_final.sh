# Final round-2 evidence: GPU tests, smoke, bench line (ours + reference arm), shares,
# the sanitizer workload run plainly, decode launch list and ncu --set full of K1f/K2w.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 300 python tools/sanitize_small.py > gpurun_out/small_workload.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 600 python tools/slab_stage.py --out gpurun_out/slab_stage.json 2>&1 | tail -6
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k_scan|k_region|k_unpack|k_plan" --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-cache --no-gather > gpurun_out/launch_bench.log 2>&1
bash tools/ncu_full.sh prof_r02c
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/small_workload.txt
