# K1 -> K2w overlap A/B: parity, strong-scaling shares, config-4 batch, full config 3.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CSVGPU_OVERLAP=0 timeout 600 python tools/slab_stage.py 2>&1 | tail -5
timeout 600 python tools/slab_stage.py 2>&1 | tail -5
CSVGPU_OVERLAP=0 timeout 300 python tools/c4_time.py 2>&1 | tail -1
timeout 300 python tools/c4_time.py 2>&1 | tail -1
for r in 1 2; do timeout 300 python tools/k2_time.py | tail -1; done
