"""Encode timing probe: repeated GPU encodes of 1024^3 timesteps next to a 34 GB resident tensor
(host-timed, synchronised), to see allocation / first-call effects on the encoder."""
import time, torch, sys
sys.path.insert(0, '.')
import paper_2308_16619_b200 as p
dev = torch.device('cuda', 0)
big = torch.empty(int(34.4e9) // 4, dtype=torch.int32, device=dev)   # like the bench's output volume
for k in range(4):
    vol = p.synth_voronoi((1024, 1024, 1024), 22, seed=3, membrane=False, drift=float(k), drift_seed=3 + k, device=dev)
    torch.cuda.synchronize()
    t = time.perf_counter()
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x = torch.empty(6 << 30, dtype=torch.uint8, device=dev); torch.cuda.synchronize()
    t2 = time.perf_counter()
    del x; torch.cuda.empty_cache()
    print(f"encode {1e3*(t1-t):.1f} ms   6GB torch alloc+free {1e3*(t2-t1):.1f} ms", flush=True)
    enc.close(); del vol; torch.cuda.empty_cache()
