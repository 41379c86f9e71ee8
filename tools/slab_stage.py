"""Single-GPU emulation of the strong-scaling decode: the config-3
volume (2048^3, 64 bz-layers) split into N whole-bz-layer shares (distributed.bz_range),
every rank's share decoded alone on this GPU (csv_decode_volume_range: the kernels a rank
runs on its own slice), timed with CUDA events (best of 3).  Projected strong-scaling
efficiency at N = full-volume time / (N * slowest share).

usage: python tools/slab_stage.py [--out profiles/r02_slab_stage.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import paper_2308_16619_b200 as p
    from paper_2308_16619_b200.distributed import bz_range
    dev = torch.device("cuda", 0)
    vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True, device=dev)
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    del vol
    torch.cuda.empty_cache()
    gv = enc.to_volume()
    out = torch.empty((2048, 2048, 2048), dtype=torch.int32, device=dev)
    res = torch.empty((gv.n_bricks, 4), dtype=torch.int64, device=dev)
    gv.set_timing(True)

    def share(z0, z1):
        best, stages = None, None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gv.decode_range(0, z0 * 4096, z1 * 4096, out[z0 * 32:z1 * 32], (z0 * 32, z1 * 32), res)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if best is None or ms < best:
                best, stages = ms, gv.last_timing()
        return best, [round(x, 3) for x in stages]

    share(0, 64)   # warm-up: workspace allocation
    full, fst = share(0, 64)
    r = {"volume": "config 3 (2048^3, 100^3 cells, membranes), 64 bz-layers", "full_ms": full,
         "full_plan_k1_k2_ms": fst, "shares": {}}
    for n in (2, 4, 8, 16, 32):
        per = []
        for rank in range(n):
            z0, z1 = bz_range(64, n, rank)
            ms, st = share(z0, z1)
            per.append({"layers": [z0, z1], "ms": round(ms, 3), "plan_k1_k2_ms": st})
        worst = max(x["ms"] for x in per)
        r["shares"][n] = {"layers_per_rank": 64 // n, "max_rank_ms": worst, "ideal_ms": full / n,
                          "projected_efficiency": full / (n * worst), "ranks": per}
        print(n, round(worst, 3), round(full / n, 3), round(full / (n * worst), 3))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(r, f, indent=1)


if __name__ == "__main__":
    main()
