"""Per-call latency of the per-brick drop-in API at LOD t = 0..5,
ours vs the reference (csvol from baseline/_ref) on the same container and bricks.

usage: python tools/brick_latency.py [--out profiles/r02_brick_latency.json] [--bricks 200]

Volume: the first 4 bz-layers (2048 x 2048 x 128 window) of config 3 (100^3 cells,
1-voxel membranes, seed 2), generated and encoded on the GPU.  Calls:
  ours  CsvContainer.decode_brick(i, t)       device-resident container, one C-ABI call
        decode_brick_entropy(...)             streams passed per call (one-brick volume per call)
  ref   csvol.CsvContainer.decode_brick(i, t) numba (JIT warmed), single thread
Each: median / p10 / p90 of per-call wall time over the same random bricks.
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def stats(ts):
    ts = sorted(ts)
    q = lambda f: ts[min(len(ts) - 1, int(f * len(ts)))]   # noqa: E731
    return {"median_us": statistics.median(ts) * 1e6, "p10_us": q(0.1) * 1e6, "p90_us": q(0.9) * 1e6, "calls": len(ts)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_brick_latency.json"))
    ap.add_argument("--bricks", type=int, default=200)
    a = ap.parse_args()
    import torch
    import paper_2308_16619_b200 as p
    dims = (2048, 2048, 128)
    vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True)[:128].contiguous()
    enc = p.compress_volume_device(vol)
    c = enc.to_container()
    enc.close()
    del vol
    rng = np.random.default_rng(3)
    idx = rng.choice(c.meta.brick_count, size=a.bricks, replace=False)
    res = {"volume": f"config-3 window {dims[0]}x{dims[1]}x{dims[2]} (first 4 bz-layers), b=32, rANS",
           "bricks": int(a.bricks), "ours": {}, "ours_streams": {}, "reference": {}}
    for i in idx[:5]:   # warm: first call uploads the container
        c.decode_brick(int(i), 0)
    for t in range(6):
        ts = []
        for i in idx:
            t0 = time.perf_counter()
            c.decode_brick(int(i), t)
            ts.append(time.perf_counter() - t0)
        res["ours"][t] = stats(ts)
        ts = []
        for i in idx[:50]:
            e = c.directory[int(i)]
            pal, co, de = c.brick_palette(int(i)), c.brick_coarse(int(i)), c.brick_detail(int(i))
            t0 = time.perf_counter()
            p.decode_brick_entropy(pal, co, int(e["coarse_nibbles"]), de, int(e["detail_nibbles"]), c.tables, t,
                                   c.config)
            ts.append(time.perf_counter() - t0)
        res["ours_streams"][t] = stats(ts)
    try:
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/csvol_numba_cache")
        import csvol
        import csvol.cli
        csvol.cli._warm_kernels()
        rc = csvol.CsvContainer.from_bytes(c.to_bytes())
        for i in idx[:3]:
            rc.decode_brick(int(i), 0)
        for t in range(6):
            ts = []
            for i in idx:
                t0 = time.perf_counter()
                ref = rc.decode_brick(int(i), t)
                ts.append(time.perf_counter() - t0)
            res["reference"][t] = stats(ts)
        # spot-check equality
        for i in idx[:20]:
            for t in (0, 1, 3):
                assert np.array_equal(rc.decode_brick(int(i), t), c.decode_brick(int(i), t))
        res["equal_checked"] = "20 bricks x t in (0, 1, 3): identical"
    except Exception as ex:   # noqa: BLE001
        res["reference"] = {"unavailable": f"{type(ex).__name__}: {ex}"}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    for t in range(6):
        r = res["reference"].get(t, {})
        print(t, round(res["ours"][t]["median_us"], 1), round(res["ours_streams"][t]["median_us"], 1),
              round(r.get("median_us", float("nan")), 1))


if __name__ == "__main__":
    main()
