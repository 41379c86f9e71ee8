"""Brick size 64 (the paper's Cortex setting) vs 32 on the config-3 field:
LOD 0 and LOD 1 full-volume decode throughput and K1 / K2 stage times (CUDA events).
N - t = 6 (b = 64, LOD 0) runs K2w<6> (final parent level in global scratch; k2_replay<6>
before, 182.7 ms -> profiles/r02_b64_before.json); LOD 1 and
every b = 32 decode run K2w.  Output: one JSON line (also written to --out).

usage: python tools/b64_probe.py [--dims 2048] [--out profiles/r02_b64.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, default=2048)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import paper_2308_16619_b200 as p
    D = a.dims
    vol = p.synth_voronoi((D, D, D), max(1, D // 20), 2, True)
    res = {"volume": f"{D}^3 Voronoi, {max(1, D // 20)}^3 cells, membranes, seed 2", "runs": []}
    for bl in (5, 6):
        enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=bl))
        gv = enc.to_volume()
        for t in (0, 1):
            cz = -(-D // (1 << t))
            out = torch.empty((cz, cz, cz), dtype=torch.int32, device="cuda")
            r = torch.empty((gv.n_bricks, 4), dtype=torch.int64, device="cuda")
            gv.decode(t, out=out, results=r)
            torch.cuda.synchronize()
            p.GpuVolume.raise_first(r, gv.n_bricks)
            gv.set_timing(True)
            ms, stages = [], []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gv.decode(t, out=out, results=r)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
                stages.append(gv.last_timing())
            gv.set_timing(False)
            best = min(range(5), key=lambda i: ms[i])
            vox = cz ** 3
            if t == 0:
                assert torch.equal(out, vol)
            res["runs"].append({"brick": 1 << bl, "lod": t, "ms": ms[best], "gvox_s": vox / (ms[best] * 1e-3) / 1e9,
                                "plan_k1_k2_ms": [round(x, 3) for x in stages[best]],
                                "k2": "k2_warp<6> (final parent level in global scratch)" if bl - t == 6 else "k2_warp<5>",
                                "compressed_bytes": enc.payload_bytes})
            del out, r
        gv.close()
        enc.close()
        torch.cuda.empty_cache()
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
