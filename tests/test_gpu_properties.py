"""SPEC acceptance properties on the GPU path, as
differential tests against the CPU oracle on seeded random inputs:

* losslessness + LOD parity on 40 seeded volumes with dims that are not multiples of
  the brick side, b in {2..64}, label patterns from smooth to noise, with and without
  rANS: GPU encode bytes == oracle encode bytes, GPU decode == input at LOD 0 and ==
  the oracle's decode at every LOD;
* rANS bit-exactness: 10^4 random nibble sequences through the batched device coder
  (csv_rans_encode / csv_rans_decode, one call each) == the oracle's scalar coder,
  and every stream decodes back."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_16619_b200 as p
    return p


def _volume(rng, kind, shape):
    z, y, x = shape
    if kind == "noise":
        return rng.integers(0, 1 << 20, size=shape, dtype=np.uint32)
    if kind == "few":
        return rng.integers(0, 3, size=shape, dtype=np.uint32)
    zz, yy, xx = np.meshgrid(np.arange(z), np.arange(y), np.arange(x), indexing="ij")
    s = int(rng.integers(2, 9))
    lab = ((xx // s) * 7 + (yy // s) * 131 + (zz // s) * 1009 + int(rng.integers(0, 1000))).astype(np.uint32)
    if kind == "membrane":
        lab = np.where((xx + 2 * yy + 3 * zz) % int(rng.integers(5, 13)) == 0, 0, lab).astype(np.uint32)
    return lab


def test_seeded_volumes_roundtrip_and_lod_parity(pkg, oracle):
    rng = np.random.default_rng(2024)
    kinds = ["smooth", "membrane", "few", "noise"]
    for case in range(40):
        bl = int(rng.integers(1, 7))
        side = 1 << bl
        shape = tuple(int(v) for v in rng.integers(1, min(3 * side, 70) + 1, size=3))
        kind = kinds[case % 4]
        entropy = bool(case % 3)
        vol = _volume(rng, kind, shape)
        ref = oracle.compress_volume(vol, brick_log2=bl, entropy=entropy)
        c = pkg.compress_volume(vol, pkg.CompressionConfig(brick_log2=bl, entropy=entropy))
        assert c.to_bytes() == ref.to_bytes(), (case, bl, shape, kind, entropy)
        assert np.array_equal(pkg.decompress_volume(c, 0), vol), (case, bl, shape, kind)
        for t in range(1, bl + 1):
            bad, _, exp = oracle.decompress_volume(ref, t)
            assert bad == -1
            assert np.array_equal(pkg.decompress_volume(c, t), exp), (case, t)


def test_rans_ten_thousand_streams(pkg, oracle):
    import torch
    from paper_2308_16619_b200 import _lib
    rng = np.random.default_rng(7)
    n = 10_000
    counts = oracle.quantize_counts(rng.integers(0, 1000, size=16))
    lens = rng.integers(0, 400, size=n).astype(np.uint32)
    p = counts / counts.sum()
    nib = [rng.choice(16, size=int(k), p=p).astype(np.uint8) for k in lens]
    offs = np.zeros(n, np.uint64)
    offs[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
    flat = np.concatenate(nib + [np.zeros(16, np.uint8)])
    boff = np.zeros(n, np.uint64)
    caps = 2 * lens.astype(np.uint64) + 8
    boff[1:] = np.cumsum(caps[:-1])
    dev = torch.device("cuda", 0)
    d_nib = torch.from_numpy(flat).to(dev)
    d_off = torch.from_numpy(offs.view(np.int64)).to(dev)
    d_len = torch.from_numpy(lens.view(np.int32)).to(dev)
    d_buf = torch.zeros(int(caps.sum()) + 16, dtype=torch.uint8, device=dev)
    d_boff = torch.from_numpy(boff.view(np.int64)).to(dev)
    d_start = torch.zeros(n, dtype=torch.int32, device=dev)
    cnt = np.ascontiguousarray(counts, dtype=np.uint16)
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.csv_rans_encode(d_nib.data_ptr(), d_off.data_ptr(), d_len.data_ptr(), n, cnt.ctypes.data,
                                 d_buf.data_ptr(), d_boff.data_ptr(), d_start.data_ptr(), s))
    buf = d_buf.cpu().numpy()
    start = d_start.cpu().numpy().view(np.uint32)
    streams = []
    for i in range(n):
        enc = buf[int(boff[i]) + int(start[i]): int(boff[i]) + int(caps[i])].tobytes()
        if i % 10 == 0:   # 10^3 byte comparisons against the oracle's scalar coder
            assert enc == oracle.rans_encode(nib[i], counts), i
        streams.append(np.frombuffer(enc, np.uint8))
    # decode all 10^4 streams in one call
    d_data = torch.from_numpy(np.concatenate(streams + [np.zeros(16, np.uint8)])).to(dev)
    soff = np.zeros(n, np.uint64)
    slen = np.array([a.size for a in streams], np.uint32)
    soff[1:] = np.cumsum(slen[:-1], dtype=np.uint64)
    d_soff = torch.from_numpy(soff.view(np.int64)).to(dev)
    d_slen = torch.from_numpy(slen.view(np.int32)).to(dev)
    d_out = torch.zeros(int(lens.sum()) + 16, dtype=torch.uint8, device=dev)
    d_status = torch.zeros(2 * n, dtype=torch.int32, device=dev)
    _lib.check(L.csv_rans_decode(d_data.data_ptr(), d_soff.data_ptr(), d_slen.data_ptr(), d_len.data_ptr(), n,
                                 cnt.ctypes.data, d_out.data_ptr(), d_off.data_ptr(), d_status.data_ptr(), s))
    st = d_status.cpu().numpy().reshape(n, 2)
    assert (st[:, 0] == 0).all()
    out = d_out.cpu().numpy()
    assert np.array_equal(out[: int(lens.sum())], flat[: int(lens.sum())])


@pytest.mark.parametrize("name", ["d_b5_mem", "a_b3", "g_b6", "c_b2_mem", "e_b4_raw"])
def test_random_corruption_matches_oracle(pkg, oracle, name):
    """150 random byte corruptions of the stream / palette sections per container
    (seeded), every brick at LOD 0-2 through the batched GPU decode (SWAR child
    evaluation, marker chains, K2w<6> for b = 64) vs the oracle's per-brick decode:
    the same (status, stream, nibble) for failures, the same labels and consumed
    counts for successes."""
    import torch
    from conftest import golden_bytes
    base = bytearray(golden_bytes(name))
    c0 = pkg.CsvContainer.from_bytes(bytes(base))
    N = c0.meta.brick_log2
    n = c0.meta.brick_count
    start = 120 + 44 * n                       # blobs follow the head and the directory
    import zlib
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    ts = [t for t in (0, 1, 2) if t < N]
    reqs = [(i, t) for i in range(n) for t in ts]
    sizes = np.array([8 ** (N - t) for _, t in reqs], dtype=np.int64)
    dst = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    bricks = torch.tensor([r[0] for r in reqs], dtype=torch.int32, device="cuda")
    lods = torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device="cuda")
    d_dst = torch.from_numpy(dst).cuda()
    pool = torch.zeros(int(sizes.sum()), dtype=torch.int32, device="cuda")
    checked = 0
    for case in range(150):
        data = bytearray(base)
        for _ in range(int(rng.integers(1, 4))):
            data[int(rng.integers(start, len(data)))] ^= int(rng.integers(1, 256))
        c = pkg.CsvContainer.from_bytes(bytes(data))
        oc = oracle.Container.from_bytes(bytes(data))
        vol = c.to_device()
        res = pkg.GpuVolume.results_host(vol.decode_bricks(bricks, lods, d_dst, pool), len(reqs))
        host = pool.cpu().numpy().view(np.uint32)
        for k, (i, t) in enumerate(reqs):
            r_ref, out_ref = oracle.container_decode_brick(oc, i, t)
            if r_ref[0] != 0:
                assert (int(res[k]["status"]), int(res[k]["stream"]), int(res[k]["pos"])) == tuple(r_ref[:3]), \
                    (name, case, i, t)
            else:
                assert int(res[k]["status"]) == 0, (name, case, i, t, res[k])
                assert (int(res[k]["ci"]), int(res[k]["di"])) == (r_ref[3], r_ref[4]), (name, case, i, t)
                assert np.array_equal(host[dst[k]: dst[k] + sizes[k]], out_ref), (name, case, i, t)
            checked += 1
        vol.close()
    assert checked == 150 * len(reqs)


@pytest.mark.parametrize("name", ["d_b5_mem", "a_b3"])
def test_overlap_plan_with_corruption_matches_oracle(pkg, oracle, name):
    """Batches of > 2048 requests take the K1 -> K2w overlap (K1 publishes finished
    bricks to a ready queue, the u8 K2w pass starts on them while K1 still runs): every
    brick at LOD 0-2, repeated until the plan is large enough, under random stream
    corruption, vs the oracle's per-brick decode (status, stream, nibble / labels and
    consumed counts)."""
    import torch
    import zlib
    from conftest import golden_bytes
    base = bytearray(golden_bytes(name))
    c0 = pkg.CsvContainer.from_bytes(bytes(base))
    N = c0.meta.brick_log2
    n = c0.meta.brick_count
    start = 120 + 44 * n
    rng = np.random.default_rng(zlib.crc32(b"ovl" + name.encode()))
    ts = [t for t in (0, 1, 2) if t < N]
    one = [(i, t) for i in range(n) for t in ts]
    reqs = one * (4200 // len(one) + 1)
    assert len(reqs) > 4096
    order = rng.permutation(len(reqs))
    reqs = [reqs[k] for k in order]
    sizes = np.array([8 ** (N - t) for _, t in reqs], dtype=np.int64)
    dst = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    bricks = torch.tensor([r[0] for r in reqs], dtype=torch.int32, device="cuda")
    lods = torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device="cuda")
    d_dst = torch.from_numpy(dst).cuda()
    pool = torch.zeros(int(sizes.sum()), dtype=torch.int32, device="cuda")
    for case in range(12):
        data = bytearray(base)
        for _ in range(int(rng.integers(0, 4)) if case else 0):
            data[int(rng.integers(start, len(data)))] ^= int(rng.integers(1, 256))
        c = pkg.CsvContainer.from_bytes(bytes(data))
        oc = oracle.Container.from_bytes(bytes(data))
        vol = c.to_device()
        res = pkg.GpuVolume.results_host(vol.decode_bricks(bricks, lods, d_dst, pool), len(reqs))
        host = pool.cpu().numpy().view(np.uint32)
        ref = {key: oracle.container_decode_brick(oc, *key) for key in one}
        for k, key in enumerate(reqs):
            r_ref, out_ref = ref[key]
            if r_ref[0] != 0:
                assert (int(res[k]["status"]), int(res[k]["stream"]), int(res[k]["pos"])) == tuple(r_ref[:3]), \
                    (name, case, key)
            else:
                assert int(res[k]["status"]) == 0, (name, case, key, res[k])
                assert (int(res[k]["ci"]), int(res[k]["di"])) == (r_ref[3], r_ref[4]), (name, case, key)
                assert np.array_equal(host[dst[k]: dst[k] + sizes[k]], out_ref), (name, case, key)
        vol.close()


def test_lod_decode_equals_independent_downsampler(pkg):
    """SPEC.md:771 / pyramid.py:99-104: for dims that are multiples of the brick side,
    the LOD-t decode of the whole volume equals the mode-of-8 downsampler applied t
    times to the input (an oracle independent of the operation replay).  The
    downsampler here is numpy, restated from pyramid.py:81-96 in the test itself."""
    def down(g):
        nz, ny, nx = g.shape
        c = g.reshape(nz // 2, 2, ny // 2, 2, nx // 2, 2).transpose(0, 2, 4, 1, 3, 5).reshape(-1, 8)
        cnt = (c[:, :, None] == c[:, None, :]).sum(axis=2)          # per slot: occurrences of its label
        win = np.argmax(cnt, axis=1)                                # first slot with the maximal count
        return c[np.arange(c.shape[0]), win].reshape(nz // 2, ny // 2, nx // 2)
    rng = np.random.default_rng(17)
    for case in range(6):
        bl = int(rng.integers(2, 6))
        side = 1 << bl
        shape = tuple(int(side * v) for v in rng.integers(1, 4, size=3))
        vol = _volume(rng, ["smooth", "membrane", "few", "noise"][case % 4], shape)
        c = pkg.compress_volume(vol, pkg.CompressionConfig(brick_log2=bl))
        ref = vol
        for t in range(bl + 1):
            if t:
                ref = down(ref)
            assert np.array_equal(pkg.decompress_volume(c, t), ref), (case, bl, shape, t)
            if t <= 2:   # the GPU downsampler (csv_downsample) agrees with the numpy one
                assert t == 0 or np.array_equal(pkg.downsample_volume(vol, t), ref), (case, t)
