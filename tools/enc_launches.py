"""One config-5 timestep encode (1024^3, 22^3 cells, seed 3) for an ncu launch list."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2308_16619_b200 as p
vol = p.synth_voronoi((1024, 1024, 1024), 22, 3, False)
for _ in range(2):
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    torch.cuda.synchronize()
    enc.close()
