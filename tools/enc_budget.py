"""Encode time of one config-5 timestep (1024^3) vs the chunk scratch budget (CSVGPU_ENC_BUDGET_GB)."""
import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2308_16619_b200 as p
vol = p.synth_voronoi((1024, 1024, 1024), 22, 3, False)
ts = []
for _ in range(int(os.environ.get("REPS", "4"))):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    enc.close()
print(os.environ.get("CSVGPU_ENC_BUDGET_GB"), [round(t, 2) for t in ts])
