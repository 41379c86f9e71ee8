# K1 A/B: parity suite on the new K1, then config-3 stage times for the new and the old kernel.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_k1.txt
timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-cache --no-gather > gpurun_out/k1_new.json 2> gpurun_out/k1_new.err
CSVGPU_K1=old timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-cache --no-gather > gpurun_out/k1_old.json 2>/dev/null
timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-cache --no-gather --zlayers 8 > gpurun_out/k1_new_z8.json 2>/dev/null
CSVGPU_K1=old timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-cache --no-gather --zlayers 8 > gpurun_out/k1_old_z8.json 2>/dev/null
cat gpurun_out/pytest_k1.txt
for f in k1_new k1_old k1_new_z8 k1_old_z8; do python -c "import json,sys;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', round(d['value'],1), d['stages_ms'], d['check'])"; done
tail -5 gpurun_out/k1_new.err
