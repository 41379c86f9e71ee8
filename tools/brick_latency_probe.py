"""Break down one per-brick call (CsvContainer.decode_brick) on the GPU box: host-side
timings of the pieces, for the latency table in DESIGN.md."""
import os, sys, time, ctypes, statistics
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16619_b200 as p
from paper_2308_16619_b200 import _lib
vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True)[:128].contiguous()
enc = p.compress_volume_device(vol)
c = enc.to_container(); enc.close(); del vol
print("max palette", int(c.directory["palette_len"].max()))
gv = c._device_volume()
def med(f, n=200):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6
s = torch.cuda.current_stream()
print("sync only", med(lambda: s.synchronize()))
x = torch.empty(1, device="cuda")
print("tiny kernel + sync", med(lambda: (x.add_(1), s.synchronize())))
out = np.empty(32768, np.uint32); res = np.zeros(1, _lib.RESULT_DTYPE)
for t in (0, 1, 4):
    b = np.array([1000], np.uint32); l = np.array([t], np.uint8)
    f = lambda: _lib.lib().csv_decode_bricks_host(gv._h, 1, b.ctypes.data, l.ctypes.data, out.ctypes.data, res.ctypes.data, s.cuda_stream)
    print("t", t, "C-ABI call", med(f), "decode_brick", med(lambda: c.decode_brick(1000, t)))
gv.set_timing(True)
for t in (0, 1, 4):
    b = np.array([1000], np.uint32); l = np.array([t], np.uint8)
    _lib.lib().csv_decode_bricks_host(gv._h, 1, b.ctypes.data, l.ctypes.data, out.ctypes.data, res.ctypes.data, s.cuda_stream)
    print("t", t, "events plan/K1/K2 ms", gv.last_timing())
