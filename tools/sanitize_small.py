"""Small decode workload for compute-sanitizer runs (memcheck / racecheck / synccheck):
config-1 container at LOD 0 and 2 (raster, K2w u8 pass), a batched Morton decode with
mixed LODs, b=64 / b=128 containers (K2w<6>, k2_replay<7>), the per-brick resident path (direct, graph capture, graph replay), the streams-per-call
scratch volume, a > 2048-request batch (K1 -> K2w overlap launch),
the rANS / pyramid drop-ins, stats() (K1 count mode), a
noise container whose palettes need the u16 K2w pass, and one device-cache frame with
LOD selection, visibility and cold-detail staging."""
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
p.decompress_volume(g, 0)                       # b=64 LOD 0: K2w<6>
with open(os.path.join(G, "vol_j_b7.csv1"), "rb") as f:
    j = p.CsvContainer.from_bytes(f.read())
p.decompress_volume(j, 0)                       # b=128 LOD 0: k2_replay<7>
p.decompress_volume(j, 1)                       # b=128 LOD 1: K2w<6>
for rep in range(3):                            # per-brick path: direct, graph capture, graph replay
    for t in (0, 1, 3):
        c.decode_brick(5 + rep, t)
e0 = c.directory[5]                             # streams passed per call: the cached scratch volume
for t in (0, 1, 3):
    p.decode_brick_entropy(c.brick_palette(5), c.brick_coarse(5), int(e0["coarse_nibbles"]), c.brick_detail(5),
                           int(e0["detail_nibbles"]), c.tables, t, c.config)
# a batch of > 2048 requests: the K1 -> K2w overlap launch (ready queue, residency guard)
nreq = 4200
ob = (torch.arange(nreq, device="cuda") % 128).to(torch.int32)
ol = (torch.arange(nreq, device="cuda") % 2).to(torch.uint8)
osz = 8 ** (5 - ol.to(torch.int64))
odst = torch.cumsum(osz, 0) - osz
opool = torch.empty(int(osz.sum()), dtype=torch.int32, device="cuda")
p.GpuVolume.raise_first(vol.decode_bricks(ob, ol, odst, opool), nreq)
tab = c.tables.leaf                             # stand-alone drop-ins
nib = np.arange(300, dtype=np.uint8) % 16
assert np.array_equal(p.rans_decode(p.rans_encode(nib, tab), 300, tab), nib)
pyr = p.build_pyramid(np.arange(4096, dtype=np.uint32) % 7, p.BrickConfig(4))
p.downsample_level(np.arange(512, dtype=np.uint32).reshape(8, 8, 8) % 5)
s = p.stats(p.CsvContainer.from_bytes(open(os.path.join(G, "vol_d_b5_mem.csv1"), "rb").read()))
k = p.CsvContainer.from_bytes(open(os.path.join(G, "vol_k_b5_noise_raw.csv1"), "rb").read())
p.decompress_volume(k, 0)
# device frame: LODs, visibility, cache assign, cold detail
import tempfile
with tempfile.TemporaryDirectory() as td:
    path = os.path.join(td, "d.csv1")
    open(path, "wb").write(open(os.path.join(G, "vol_d_b5_mem.csv1"), "rb").read())
    cold = p.CsvContainer.open(path, detail_cold=True)
    cv = cold.to_device()
    lods = p.desired_lods_device(cv, p.Camera(position=(0.0, 0.0, 0.0), height=64))
    vis = p.visibility_mask_device(cv, p.TransferFunction(0.0, {0: (1.0, 1.0, 1.0, 1.0)}))
    nb = cold.meta.brick_count
    cache = p.DeviceBrickCache(nb, 5, pool_bytes=nb * 8 ** 4 * 32 + 4096)
    ds = p.DeviceDetailStream(cold, cv, budget_bytes=4096)
    cache.begin_frame()
    req = [(i, 0) for i in range(nb)]
    cache.mark_used([r[0] for r in req], [0] * nb)
    adj = ds.plan(req)
    cache.end_frame_assign([a[0] for a in adj], [a[1] for a in adj], cv, detail=ds)
    cache.close()
    cv.close()
torch.cuda.synchronize()
print("sanitize workload ok", s["total_ops"])
