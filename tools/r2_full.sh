# Full GPU evidence pass: parity, smoke, bench (ours + reference arm), decode launch list,
# ncu --set full of K1f + K2w, strong-scaling emulation, b=64 probe, per-brick latency.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k_scan|k_region|k_plan|k_unpack" --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-cache --no-gather > gpurun_out/launch_bench.log 2>&1
bash tools/ncu_full.sh prof_full
timeout 900 python tools/slab_stage.py --out gpurun_out/slab_stage.json > gpurun_out/slab_stage.txt 2>&1
timeout 900 python tools/b64_probe.py --out gpurun_out/b64.json > /dev/null 2>&1
timeout 900 python tools/brick_latency.py --out gpurun_out/brick_latency.json > gpurun_out/brick_latency.txt 2>&1
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/slab_stage.txt gpurun_out/brick_latency.txt
python -c "import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(d['value'], d['stages_ms'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
