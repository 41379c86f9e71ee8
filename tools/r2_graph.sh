# Per-brick graph path: parity tests, latency table graph off/on, then the decode evidence (launch list + ncu).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CSVGPU_BRICK_GRAPH=0 timeout 600 python tools/brick_latency.py --out gpurun_out/lat_nograph.json 2>&1 | tail -7
timeout 600 python tools/brick_latency.py --out gpurun_out/lat_graph.json 2>&1 | tail -7
bash tools/r2_prof.sh
