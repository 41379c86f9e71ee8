"""Config-4 (65,536 nearest bricks, mixed LOD 0/1) batched decode: per-stage timing."""
import json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2308_16619_b200 as p
from bench import desired_lods

dev = torch.device("cuda", 0)
vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True, device=dev)
enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
del vol
torch.cuda.empty_cache()
gx = gy = gz = 64
lod, dist = desired_lods((gx, gy, gz), 32, (1024.0, 1024.0, -64.0), math.pi / 3, 1080, 5)
order = np.argsort(dist, kind="stable")[:65536]
reqs = [(int(i), int(lod[i])) for i in order if lod[i] < 5]
sizes = np.array([8 ** (5 - l) for _, l in reqs], dtype=np.int64)
dst = np.concatenate([[0], np.cumsum(sizes)[:-1]])
pool = torch.empty(int(sizes.sum()), dtype=torch.int32, device=dev)
full = enc.to_volume()
b = torch.tensor([r[0] for r in reqs], dtype=torch.int32, device=dev)
l = torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device=dev)
d = torch.from_numpy(dst).to(dev)
res = torch.empty((len(reqs), 4), dtype=torch.int64, device=dev)
full.decode_bricks(b, l, d, pool, results=res)
full.set_timing(True)
ts = []
for _ in range(5):
    full.decode_bricks(b, l, d, pool, results=res)
    torch.cuda.synchronize()
    ts.append(full.last_timing())
ts.sort(key=lambda x: sum(x))
m = ts[2]
vox = int(sizes.sum())
print(json.dumps({"plan": round(m[0], 3), "k1": round(m[1], 3), "k2": round(m[2], 3),
                  "gvox_s": round(vox / (sum(m) * 1e6), 1), "lib": os.environ.get("CSVGPU_LIB", "default")}))
