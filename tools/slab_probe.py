"""Decode config 3 whole vs in z-slabs of k bz-layers (same stream): does K1->K2 locality help?"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16619_b200 as p

dev = torch.device("cuda", 0)
vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True, device=dev)
enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
del vol
torch.cuda.empty_cache()
gv = enc.to_volume((0, 64 * 64 * 64))
out = torch.empty((2048, 2048, 2048), dtype=torch.int32, device=dev)
res = torch.empty((gv.n_bricks, 4), dtype=torch.int64, device=dev)
gv.decode(0, out=out, results=res)
torch.cuda.synchronize()
ref = out[::64, ::64, ::64].clone()
r = {}
for layers in (64, 16, 8, 4, 2, 1):
    per = 64 * 64 * layers
    def run():
        for z in range(0, 64, layers):
            gv.decode_range(0, z * 64 * 64, (z + layers) * 64 * 64, out[z * 32:(z + layers) * 32],
                            (z * 32, (z + layers) * 32), res)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        run()
    e1.record()
    torch.cuda.synchronize()
    r[layers] = round(e0.elapsed_time(e1) / 3, 3)
    assert torch.equal(out[::64, ::64, ::64], ref)
print(json.dumps(r))
