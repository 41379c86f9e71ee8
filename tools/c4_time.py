"""Config-4 batched decode (65,536 requests, Morton pool): stage times (CUDA events)."""
import math, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2308_16619_b200 as p
import bench
vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True)
enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
del vol; torch.cuda.empty_cache()
lod, dist = bench.desired_lods((64, 64, 64), 32, (1024.0, 1024.0, -64.0), math.pi / 3, 1080, 5)
order = np.argsort(dist, kind="stable")[:65536]
reqs = [(int(i), int(lod[i])) for i in order if lod[i] < 5]
sizes = np.array([8 ** (5 - t) for _, t in reqs], dtype=np.int64)
dst = np.concatenate([[0], np.cumsum(sizes)[:-1]])
gv = enc.to_volume()
pool = torch.empty(int(sizes.sum()), dtype=torch.int32, device="cuda")
b = torch.tensor([r[0] for r in reqs], dtype=torch.int32, device="cuda")
l = torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device="cuda")
d = torch.from_numpy(dst).cuda()
res = torch.empty((len(reqs), 4), dtype=torch.int64, device="cuda")
gv.decode_bricks(b, l, d, pool, results=res)
gv.set_timing(True)
st = []
for _ in range(5):
    gv.decode_bricks(b, l, d, pool, results=res)
    st.append(gv.last_timing())
t = [min(s[i] for s in st) for i in range(3)]
print("config4 plan/K1/K2 ms", [round(x, 3) for x in t], "GVox/s", round(int(sizes.sum()) / (sum(t) * 1e-3) / 1e9, 1))
