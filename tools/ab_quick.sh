# config-3 stage times for the in-tree build and every variants/*.so (no parity run)
for so in paper_2308_16619_b200/libcsvgpu.so variants/*.so; do
  CSVGPU_LIB=$PWD/$so timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --no-cache --no-gather > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]);print('$so', round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()}, d['check']['mismatches'])" || tail -3 /tmp/ab.err
done
