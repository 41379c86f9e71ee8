"""Where the host-in / host-out decode (decompress_volume) spends its time on config 3:
volume creation + close (device allocations) vs the slab pipeline, five calls in a row."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_16619_b200 as p  # noqa: E402
from paper_2308_16619_b200.device import GpuVolume  # noqa: E402

dev = torch.device("cuda", 0)
vol = p.synth_voronoi((2048, 2048, 2048), 2048 // 100 + 1, 2, True, device=dev)
enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
cont = enc.to_container()
enc.close()
del vol
torch.cuda.empty_cache()
pin = torch.empty((2048, 2048, 2048), dtype=torch.int32, pin_memory=True)
pn = pin.numpy().view(np.uint32)
d = cont.directory
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gv = GpuVolume(cont.head_bytes(), d, cont.palette_blob.size, cont.coarse_blob.size, cont.detail_blob.size,
                   deferred=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    gv.close()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    p.decompress_volume(cont, 0, out=pn)
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  close {1e3*(t2-t1):.1f} ms  decompress_volume {1e3*(t3-t2):.1f} ms", flush=True)
