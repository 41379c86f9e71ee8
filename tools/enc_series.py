"""Config-5 encode timing per timestep as bench.py's timeseries leg runs it (synth, encode,
decode, close, empty_cache), with CSVGPU_ENC_TRACE phase times for investigations."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2308_16619_b200 as p
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
res = []
for k in range(int(os.environ.get("STEPS", "8"))):
    vol = p.synth_voronoi((1024, 1024, 1024), 22, seed=3, membrane=False, drift=float(min(k, 16)), drift_seed=3 + k,
                          device=dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    e1.record(stream)
    torch.cuda.synchronize()
    host = (time.perf_counter() - t0) * 1e3
    print(f"step {k}: encode {e0.elapsed_time(e1):.2f} ms (host {host:.2f})", file=sys.stderr, flush=True)
    res.append(round(e0.elapsed_time(e1), 2))
    gv = enc.to_volume()
    out = torch.empty_like(vol)
    gv.decode(0, out=out)
    torch.cuda.synchronize()
    gv.close()
    enc.close()
    del vol, out
    if os.environ.get("EMPTY", "1") == "1":
        torch.cuda.empty_cache()
print(res)
