# Final round-2 evidence: GPU tests, smoke, bench line (ours + reference arm), shares, sanitizer on the small paths.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 600 python tools/slab_stage.py --out gpurun_out/slab_stage.json 2>&1 | tail -6
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt
