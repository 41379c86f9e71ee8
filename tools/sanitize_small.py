"""Small decode workload for compute-sanitizer runs (memcheck / racecheck / synccheck):
config-1 container at LOD 0 and 2 (raster), a batched Morton decode with mixed LODs,
a b=64 container (global-workspace kernel) and stats() (K1 count mode)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_16619_b200 as p  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
with open(os.path.join(G, "config1.csv1"), "rb") as f:
    c = p.CsvContainer.from_bytes(f.read())
vol = c.to_device(brick_range=(0, 128))
for t in (0, 2):
    p.decompress_volume_device(vol, t)
bricks = torch.arange(0, 64, dtype=torch.int32, device="cuda")
lods = (torch.arange(0, 64, device="cuda") % 3).to(torch.uint8)
sizes = (8 ** (5 - lods.to(torch.int64)))
dst = torch.cumsum(sizes, 0) - sizes
pool = torch.empty(int(sizes.sum()), dtype=torch.int32, device="cuda")
p.GpuVolume.raise_first(vol.decode_bricks(bricks, lods, dst, pool), 64)
with open(os.path.join(G, "vol_g_b6.csv1"), "rb") as f:
    g = p.CsvContainer.from_bytes(f.read())
p.decompress_volume(g, 0)
s = p.stats(p.CsvContainer.from_bytes(open(os.path.join(G, "vol_d_b5_mem.csv1"), "rb").read()))
torch.cuda.synchronize()
print("sanitize workload ok", s["total_ops"])
