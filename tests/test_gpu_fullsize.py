"""Full-size properties (BASELINE.json configs 2/3 shapes) on the B200: encode -> decode
round trip is lossless for every voxel of a 2048^3 volume, sampled bricks at LOD 0/1/2
decode exactly like the CPU oracle, the device brick cache reproduces the raster decode,
and the raster LOD-t decode equals the Morton decode of every brick (checksummed)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def big():
    import torch
    import paper_2308_16619_b200 as p
    dev = torch.device("cuda", 0)
    vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True, device=dev)     # config 3 input
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    yield p, torch, vol, enc
    del vol, enc
    torch.cuda.empty_cache()


def test_config3_lossless_roundtrip(big):
    p, torch, vol, enc = big
    gv = enc.to_volume()
    out, res = gv.decode(0)
    p.GpuVolume.raise_first(res, gv.n_bricks)
    for z0 in range(0, 2048, 256):                 # compare in slabs (bounded temporaries)
        assert torch.equal(out[z0:z0 + 256], vol[z0:z0 + 256]), z0
    del out


def test_config3_sampled_bricks_match_oracle(big, oracle):
    p, torch, vol, enc = big
    cont = enc.to_container()
    oc = oracle.Container.from_bytes(cont.to_bytes())
    rng = np.random.default_rng(7)
    bricks = rng.choice(64 ** 3, size=48, replace=False)
    gv = enc.to_volume()
    reqs = [(int(b), t) for b in bricks for t in (0, 1, 2)]
    sizes = np.array([8 ** (5 - t) for _, t in reqs], dtype=np.int64)
    dst = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    pool = torch.zeros(int(sizes.sum()), dtype=torch.int32, device="cuda")
    res = gv.decode_bricks(torch.tensor([r[0] for r in reqs], dtype=torch.int32, device="cuda"),
                           torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device="cuda"),
                           torch.from_numpy(dst).cuda(), pool)
    p.GpuVolume.raise_first(res, len(reqs))
    host = pool.cpu().numpy().view(np.uint32)
    for k, (b, t) in enumerate(reqs):
        bad, ref = oracle.container_decode_brick(oc, b, t)
        assert np.array_equal(host[dst[k]: dst[k] + sizes[k]], ref), (b, t)


def test_config3_lod1_raster_equals_morton_bricks(big):
    """Raster LOD-1 decode of the whole volume == per-brick Morton decodes placed by
    morton_to_grid (a size-independent consistency check of K3 vs K4)."""
    p, torch, vol, enc = big
    gv = enc.to_volume()
    out, res = gv.decode(1)
    p.GpuVolume.raise_first(res, gv.n_bricks)
    side = 16
    rng = np.random.default_rng(3)
    bricks = rng.choice(64 ** 3, size=64, replace=False)
    pool = torch.zeros(len(bricks) * side ** 3, dtype=torch.int32, device="cuda")
    dst = torch.arange(len(bricks), dtype=torch.int64, device="cuda") * side ** 3
    res = gv.decode_bricks(torch.tensor(bricks, dtype=torch.int32, device="cuda"),
                           torch.ones(len(bricks), dtype=torch.uint8, device="cuda"), dst, pool)
    p.GpuVolume.raise_first(res, len(bricks))
    from paper_2308_16619_b200.morton import morton_encode
    m = torch.tensor([[[morton_encode(int(x), int(y), int(z)) for x in range(side)] for y in range(side)]
                      for z in range(side)], dtype=torch.int64, device="cuda")
    for k, b in enumerate(bricks.tolist()):
        bx, by, bz = b % 64, (b // 64) % 64, b // 4096
        brick = pool[k * side ** 3:(k + 1) * side ** 3][m]
        assert torch.equal(brick, out[bz * side:(bz + 1) * side, by * side:(by + 1) * side, bx * side:(bx + 1) * side]), b


def test_config4_exact_batch_matches_oracle(big, oracle):
    """Config 4 exactly as bench.py runs it: camera (1024, 1024, -64) +z, H=1080,
    fov pi/3, desired_lods, the 65,536 nearest bricks -> BrickCache plan -> ONE
    batched csv_decode_bricks into the 8 GiB pool.  Every request must succeed;
    96 sampled placements (both LODs) are compared with the oracle."""
    import math
    import bench
    p, torch, vol, enc = big
    gx = gy = gz = 64
    lod, dist = bench.desired_lods((gx, gy, gz), 32, (1024.0, 1024.0, -64.0), math.pi / 3, 1080, 5)
    order = np.argsort(dist, kind="stable")[:65536]
    reqs = [(int(i), int(lod[i])) for i in order if lod[i] < 5]
    assert len(reqs) == 65536
    cache = p.BrickCache(gx * gy * gz, 5, pool_bytes=8 << 30, device=torch.device("cuda", 0))
    cache.begin_frame()
    for br, l in reqs:
        cache.mark_used(br, l)
    placed, live = cache.plan_frame(reqs)
    arr = np.asarray(live, dtype=np.int64)
    assert len(arr) == 65536 and {int(x) for x in arr[:, 1]} == {0, 1}
    gv = enc.to_volume()
    res = gv.decode_bricks(torch.from_numpy(arr[:, 0].astype(np.int32)).cuda(),
                           torch.from_numpy(arr[:, 1].astype(np.uint8)).cuda(),
                           torch.from_numpy(arr[:, 2] * 8).cuda(), cache.pool)
    p.GpuVolume.raise_first(res, len(arr))
    assert int((res[:len(arr), 0] & 0xFFFFFFFF).ne(0).sum()) == 0
    oc = oracle.Container.from_bytes(enc.to_container().to_bytes())
    rng = np.random.default_rng(11)
    pick = np.concatenate([rng.choice(np.flatnonzero(arr[:, 1] == t), size=48, replace=False) for t in (0, 1)])
    pool = cache.pool
    for k in pick:
        b, t, start = (int(v) for v in arr[k, :3])
        n = 8 ** (5 - t)
        got = pool[start * 8: start * 8 + n].cpu().numpy().view(np.uint32)
        _, ref = oracle.container_decode_brick(oc, b, t)
        assert np.array_equal(got, ref), (b, t)


@pytest.fixture()
def config2():
    import torch
    import paper_2308_16619_b200 as p
    dev = torch.device("cuda", 0)
    vol = p.synth_voronoi((1024, 1024, 1024), 22, 1, False, device=dev)     # config 2 input
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
    yield p, torch, vol, enc
    enc.close()
    del vol
    torch.cuda.empty_cache()


def test_config2_lossless_and_sampled_bricks(config2, oracle):
    """Config 2 (1024^3, ~10k labels): the full LOD-0 decode equals the input voxel for
    voxel; 48 sampled bricks at LOD 0-2 equal the oracle's decode of the same container."""
    p, torch, vol, enc = config2
    gv = enc.to_volume()
    out, res = gv.decode(0)
    p.GpuVolume.raise_first(res, gv.n_bricks)
    assert torch.equal(out, vol)
    del out
    oc = oracle.Container.from_bytes(enc.to_container().to_bytes())
    rng = np.random.default_rng(5)
    bricks = rng.choice(32 ** 3, size=48, replace=False)
    reqs = [(int(b), t) for b in bricks for t in (0, 1, 2)]
    sizes = np.array([8 ** (5 - t) for _, t in reqs], dtype=np.int64)
    dst = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    pool = torch.zeros(int(sizes.sum()), dtype=torch.int32, device="cuda")
    res = gv.decode_bricks(torch.tensor([r[0] for r in reqs], dtype=torch.int32, device="cuda"),
                           torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device="cuda"),
                           torch.from_numpy(dst).cuda(), pool)
    p.GpuVolume.raise_first(res, len(reqs))
    host = pool.cpu().numpy().view(np.uint32)
    for k, (b, t) in enumerate(reqs):
        _, ref = oracle.container_decode_brick(oc, b, t)
        assert np.array_equal(host[dst[k]: dst[k] + sizes[k]], ref), (b, t)


def test_config5_two_timesteps_roundtrip(oracle):
    """Config 5's per-GPU share: two 1024^3 timesteps with drifting seeds (seed 3, drift
    0 and 1 voxel), encoded and decoded on the GPU: lossless; the first bz-layer of
    each timestep encodes byte-identically to the oracle's compress_volume."""
    import torch
    import paper_2308_16619_b200 as p
    dev = torch.device("cuda", 0)
    for k in range(2):
        vol = p.synth_voronoi((1024, 1024, 1024), 22, 3, False, drift=float(k), drift_seed=3 + k, device=dev)
        enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
        gv = enc.to_volume()
        out, res = gv.decode(0)
        p.GpuVolume.raise_first(res, gv.n_bricks)
        assert torch.equal(out, vol), k
        layer = vol[:32].contiguous()
        mine = p.compress_volume_device(layer, p.CompressionConfig(brick_log2=5)).to_container().to_bytes()
        ref = oracle.compress_volume(layer.cpu().numpy().view(np.uint32), brick_log2=5).to_bytes()
        assert mine == ref, k
        gv.close()
        enc.close()
        del vol, out, layer
        torch.cuda.empty_cache()
