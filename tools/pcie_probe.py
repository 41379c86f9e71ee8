import torch, time
dev = torch.device("cuda")
n = 1 << 30  # 4 GB of int32
d = torch.empty(n, dtype=torch.int32, device=dev)
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); print("D2H 1 stream", 4 / (t1 - t0), "GB/s")
    ss = [torch.cuda.Stream() for _ in range(4)]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for i, s in enumerate(ss):
        with torch.cuda.stream(s):
            h[i * n // 4:(i + 1) * n // 4].copy_(d[i * n // 4:(i + 1) * n // 4], non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter(); print("D2H 4 streams", 4 / (t1 - t0), "GB/s")
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); print("H2D pinned", 4 / (t1 - t0), "GB/s")
    import numpy as np
    a = np.ones(n // 4, dtype=np.int32)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d[: n // 4].copy_(torch.from_numpy(a)); torch.cuda.synchronize()
    t1 = time.perf_counter(); print("H2D pageable", 1 / (t1 - t0), "GB/s")
