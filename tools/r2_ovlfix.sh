# Overlap-launch residency guard: GPU tests x3 (the overlap+corruption test was flaky), shares, config-4 batch.
set -x
mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt_$i.txt 2>&1; tail -1 gpurun_out/pt_$i.txt; done
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_properties.py -m gpu -x -q -k overlap 2>&1 | tail -1; done
timeout 600 python tools/slab_stage.py 2>&1 | tail -6
timeout 300 python tools/c4_time.py 2>&1 | tail -1
