"""The K1 floor of a strong-scaling share: the longest rANS stream of config 3 and how
long one lane takes for it alone (per-brick call at t = 0, CUDA-event stage times).
usage: python tools/stream_floor.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2308_16619_b200 as p
    vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True)
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    del vol
    torch.cuda.empty_cache()
    c = enc.to_container()
    enc.close()
    d = c.directory
    dn = d["detail_nibbles"].astype(np.int64)
    cn = d["coarse_nibbles"].astype(np.int64)
    order = np.argsort(-dn)
    print("detail nibbles: max %d  p99.9 %d  p99 %d  median %d  mean %.0f" %
          (dn.max(), np.percentile(dn, 99.9), np.percentile(dn, 99), np.median(dn), dn.mean()))
    print("coarse nibbles: max %d  median %d" % (cn.max(), np.median(cn)))
    gv = c._device_volume()
    gv.set_timing(True)
    for i in order[:3]:
        for rep in range(3):
            t0 = time.perf_counter()
            c.decode_brick(int(i), 0)
            wall = (time.perf_counter() - t0) * 1e6
        ms = gv.last_timing()
        print("brick %d: %d detail nibbles, call %.0f us, stages %s, %.1f ns per symbol (K1)" %
              (i, dn[i], wall, [round(x, 3) for x in ms], ms[1] * 1e6 / dn[i]))


if __name__ == "__main__":
    main()
