import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2308_16619_b200 as p
dev = torch.device("cuda", 0)
vol = p.synth_voronoi((2048, 2048, 64), 100, 2, True, device=dev)
enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
gv = enc.to_volume((0, 64 * 64 * 2))
out = torch.empty((64, 2048, 2048), dtype=torch.int32, device=dev)
res = torch.empty((gv.n_bricks, 4), dtype=torch.int64, device=dev)
for _ in range(2):
    gv.decode_range(0, 0, 4096, out[:32], (0, 32), res)
torch.cuda.synchronize()
print("ok")
