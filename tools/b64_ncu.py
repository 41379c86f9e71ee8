"""b = 64 config-3 field decoded once at LOD 0 (for an ncu capture of K2w<6>)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2308_16619_b200 as p
vol = p.synth_voronoi((2048, 2048, 2048), 102, 2, True)
enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=6))
del vol
torch.cuda.empty_cache()
gv = enc.to_volume()
out = torch.empty((2048, 2048, 2048), dtype=torch.int32, device="cuda")
for _ in range(2):
    gv.decode(0, out=out)
torch.cuda.synchronize()
