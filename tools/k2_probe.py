"""Per-stage decode timing of the config-3 volume at several LODs (kernel A/B tool).

usage: CSVGPU_LIB=path/to/variant.so python tools/k2_probe.py [--zlayers K] [--lods 0,1,2] [--reps 5]
Prints one JSON line: per LOD the median plan/K1/K2 milliseconds and an output
checksum (so variants can be compared for identical results).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--zlayers", type=int, default=64)
    ap.add_argument("--lods", default="0,1,2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cells", type=int, default=100)
    ap.add_argument("--membrane", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2308_16619_b200 as p
    dev = torch.device("cuda", 0)
    dims = (2048, 2048, 32 * a.zlayers)
    vol = p.synth_voronoi(dims, a.cells, 2, bool(a.membrane), device=dev)
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    del vol
    torch.cuda.empty_cache()
    gv = enc.to_volume((0, 64 * 64 * a.zlayers))
    res = {"lib": os.environ.get("CSVGPU_LIB", "default"), "zlayers": a.zlayers}
    for t in map(int, a.lods.split(",")):
        out, r = gv.decode(t)
        p.GpuVolume.raise_first(r, gv.n_bricks)
        ck = 0
        flat = out.view(-1)
        for c0 in range(0, flat.numel(), 1 << 28):
            v = flat[c0:c0 + (1 << 28)].to(torch.int64)
            w = (torch.arange(v.numel(), device=dev, dtype=torch.int64) + c0) % 1000003
            ck = (ck + int(((v * w) % (1 << 61)).sum().item())) % (1 << 61)
            del v, w
        gv.set_timing(True)
        st = []
        for _ in range(a.reps):
            gv.decode(t, out=out, results=r)
            torch.cuda.synchronize()
            st.append(gv.last_timing())
        gv.set_timing(False)
        st.sort(key=lambda s: s[1] + s[2])
        m = st[len(st) // 2]
        vox = out.numel()
        res[f"t{t}"] = {"plan": round(m[0], 3), "k1": round(m[1], 3), "k2": round(m[2], 3),
                        "gvox_s": round(vox / ((m[0] + m[1] + m[2]) * 1e6), 1), "ck": ck}
        del out, r
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
