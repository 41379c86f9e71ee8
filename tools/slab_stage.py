import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
import paper_2308_16619_b200 as p
dev = torch.device("cuda", 0)
vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True, device=dev)
enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
del vol; torch.cuda.empty_cache()
gv = enc.to_volume((0, 64 * 64 * 64))
out = torch.empty((2048, 2048, 2048), dtype=torch.int32, device=dev)
res = torch.empty((gv.n_bricks, 4), dtype=torch.int64, device=dev)
gv.set_timing(True)
r = {}
for layers in (64, 8, 1):
    ts = []
    for rep in range(3):
        z = 0
        gv.decode_range(0, z * 4096, (z + layers) * 4096, out[z*32:(z+layers)*32], (z*32, (z+layers)*32), res)
        torch.cuda.synchronize()
        ts.append(gv.last_timing())
    r[layers] = [round(x, 3) for x in ts[-1]]
print(json.dumps(r))
