"""GPU parity: the sm_100a decode path (C-ABI -> K1/K2) vs the reference's golden outputs
and the CPU oracle.  Bit-exact for every label; error messages byte-identical."""
import hashlib

import numpy as np
import pytest

from conftest import FUZZ, VOLUMES, GOLDEN, fuzz_container_bytes, golden_bytes, golden_json, golden_volume, h16

pytestmark = pytest.mark.gpu

COLS = {"palette_off": 0, "palette_len": 1, "coarse_off": 2, "coarse_bytes": 3, "coarse_nibbles": 4,
        "detail_off": 5, "detail_bytes": 6, "detail_nibbles": 7}


@pytest.fixture(scope="module")
def pkg():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_16619_b200 as p
    return p


@pytest.mark.parametrize("name", VOLUMES)
def test_decompress_volume_all_lods(pkg, name):
    g = golden_json(f"decode_{name}.json")
    c = pkg.CsvContainer.from_bytes(golden_bytes(name))
    for t in range(g["brick_log2"] + 1):
        vol = pkg.decompress_volume(c, t)
        assert h16(vol) == g["volume"][str(t)], (name, t)
    vol = pkg.decompress_volume(c, 0)
    assert np.array_equal(vol, golden_volume(name).astype(np.uint32))


@pytest.mark.parametrize("name", VOLUMES)
def test_batched_bricks_all_lods(pkg, name):
    """K4: every (brick, t) of the volume in one batch, Morton order, consumed counts."""
    import torch
    g = golden_json(f"decode_{name}.json")
    c = pkg.CsvContainer.from_bytes(golden_bytes(name))
    N = g["brick_log2"]
    vol = c.to_device()
    reqs = [(int(i), t) for i in g["bricks"] for t in range(N + 1)]
    sizes = [8 ** (N - t) for _, t in reqs]
    dst = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    # keep 16-byte alignment for most, but exercise unaligned destinations too
    pool = torch.zeros(int(sum(sizes)) + 8, dtype=torch.int32, device="cuda")
    bricks = torch.tensor([r[0] for r in reqs], dtype=torch.int32, device="cuda")
    lods = torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device="cuda")
    res = vol.decode_bricks(bricks, lods, torch.from_numpy(dst).cuda(), pool)
    rh = pkg.GpuVolume.results_host(res, len(reqs))
    host = pool.cpu().numpy().view(np.uint32)
    for k, (i, t) in enumerate(reqs):
        exp = g["bricks"][str(i)][str(t)]
        out = host[dst[k]: dst[k] + sizes[k]]
        assert rh[k]["status"] == 0
        if t < N:
            assert [h16(out), int(rh[k]["ci"]), int(rh[k]["di"])] == exp[1:], (name, i, t)
        else:
            assert h16(out) == exp[1]


@pytest.mark.parametrize("name", ["a_b3", "d_b5_mem", "e_b4_raw", "g_b6"])
def test_decode_brick_api(pkg, name):
    """CsvContainer.decode_brick / decode_brick_entropy(return_consumed) single-brick API."""
    g = golden_json(f"decode_{name}.json")
    c = pkg.CsvContainer.from_bytes(golden_bytes(name))
    N = g["brick_log2"]
    for i in list(g["bricks"])[:4]:
        for t in range(N + 1):
            out = c.decode_brick(int(i), t)
            assert h16(out) == g["bricks"][i][str(t)][1]
    if c.meta.entropy:
        i = 0
        e = c.directory[i]
        out, ci, di = pkg.decode_brick_entropy(c.brick_palette(i), c.brick_coarse(i), int(e["coarse_nibbles"]),
                                               c.brick_detail(i), int(e["detail_nibbles"]), c.tables, 0, c.config,
                                               return_consumed=True)
        assert [h16(out), ci, di] == g["bricks"]["0"]["0"][1:]


def _gpu_outcome(pkg, c, i, t):
    try:
        out = c.decode_brick(i, t)
    except pkg.CorruptStreamError as e:
        return ["err", str(e)]
    return ["ok", h16(out)]


@pytest.mark.parametrize("name", FUZZ)
def test_fuzz_error_parity(pkg, name):
    """Corrupted streams: same exception text (status, stream, nibble) or same labels."""
    import torch
    base = golden_bytes(name)
    cases = golden_json(f"fuzz_{name}.json")
    for case in cases:
        c = pkg.CsvContainer.from_bytes(fuzz_container_bytes(base, case))
        if case["dir"]:
            d = c.directory.copy()
            d[case["brick"]][case["dir"][0]] = case["dir"][1]
            c.directory = d
        vol = c.to_device()
        ts = [int(t) for t in case["outcomes"]]
        n = len(ts)
        N = c.meta.brick_log2
        sizes = [8 ** (N - t) for t in ts]
        dst = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
        pool = torch.zeros(int(sum(sizes)), dtype=torch.int32, device="cuda")
        res = vol.decode_bricks(torch.full((n,), case["brick"], dtype=torch.int32, device="cuda"),
                                torch.tensor(ts, dtype=torch.uint8, device="cuda"),
                                torch.from_numpy(dst).cuda(), pool)
        rh = pkg.GpuVolume.results_host(res, n)
        host = pool.cpu().numpy().view(np.uint32)
        from paper_2308_16619_b200.device import status_error
        for k, t in enumerate(ts):
            exp = case["outcomes"][str(t)]
            if rh[k]["status"] != 0:
                got = ["err", str(status_error(int(rh[k]["status"]), int(rh[k]["stream"]), int(rh[k]["pos"])))]
            else:
                got = ["ok", h16(host[dst[k]: dst[k] + sizes[k]]), int(rh[k]["ci"]), int(rh[k]["di"])]
            assert got == exp, (name, case, t)


@pytest.mark.parametrize("name", ["d_b5_mem", "e_b4_raw"])
def test_fuzz_resident_decode_brick(pkg, name):
    """CsvContainer.decode_brick on the device-resident container (csv_decode_bricks_host)
    raises the reference's exact message, or returns its labels, for corrupted streams."""
    base = golden_bytes(name)
    for case in golden_json(f"fuzz_{name}.json")[:80]:
        c = pkg.CsvContainer.from_bytes(fuzz_container_bytes(base, case))
        if case["dir"]:
            d = c.directory.copy()
            d[case["brick"]][case["dir"][0]] = case["dir"][1]
            c.directory = d
        for t, exp in case["outcomes"].items():
            assert _gpu_outcome(pkg, c, case["brick"], int(t)) == exp[:2], (name, case, t)


@pytest.mark.parametrize("name", ["d_b5_mem", "g_b6", "h_b3_u16"])
def test_resident_graph_replay(pkg, oracle, name):
    """Per-brick calls on one device-resident container: the first call of a (requests,
    voxels) shape launches directly, the second captures the CUDA graph, later ones replay
    it (the request copy reads the pinned staging at replay time; labels and results land
    in mapped pinned memory).  Three passes over every brick at every LOD, bricks in a
    shuffled order, each call vs the oracle; then a corrupted directory entry (new
    container) raises the reference's message on the replayed path as well."""
    data = golden_bytes(name)
    c = pkg.CsvContainer.from_bytes(data)
    oc = oracle.Container.from_bytes(data)
    N = c.meta.brick_log2
    n = c.meta.brick_count
    rng = np.random.default_rng(11)
    ref = {}
    for rep in range(3):
        for t in range(N):   # (t == N is palette[0], no decode)
            for i in rng.permutation(n)[: min(n, 24)]:
                i = int(i)
                if (i, t) not in ref:
                    ref[(i, t)] = oracle.container_decode_brick(oc, i, t)[1]
                assert np.array_equal(c.decode_brick(i, t), ref[(i, t)]), (name, rep, i, t)
    d = c.directory.copy()
    d[1]["coarse_bytes"] = 2   # truncated coarse stream
    c2 = pkg.CsvContainer.from_bytes(data)
    c2.directory = d
    oc2 = oracle.Container.from_bytes(data)
    oc2.directory[1, 3] = 2   # DIR_COLS[3] == coarse_bytes
    bad, _ = oracle.container_decode_brick(oc2, 1, 1)
    assert bad[0] != 0
    msgs = set()
    for _ in range(4):   # direct, capture, replay, replay
        with pytest.raises(pkg.CorruptStreamError) as ei:
            c2.decode_brick(1, 1)
        msgs.add(str(ei.value))
        assert np.array_equal(c2.decode_brick(0, 1), oracle.container_decode_brick(oc, 0, 1)[1])
    from paper_2308_16619_b200.device import status_error
    assert msgs == {str(status_error(*bad[:3]))}


def test_resident_decode_brick_threads(pkg, oracle):
    """decode_brick from four Python threads on one container (ctypes drops the GIL; the
    per-volume staging and graphs are serialised in csv_decode_bricks_host)."""
    import threading
    data = golden_bytes("d_b5_mem")
    c = pkg.CsvContainer.from_bytes(data)
    oc = oracle.Container.from_bytes(data)
    n = c.meta.brick_count
    ref = {(i, t): oracle.container_decode_brick(oc, i, t)[1] for i in range(n) for t in (0, 1, 2)}
    bad = []

    def work(seed):
        rng = np.random.default_rng(seed)
        for _ in range(60):
            i, t = int(rng.integers(n)), int(rng.integers(3))
            if not np.array_equal(c.decode_brick(i, t), ref[(i, t)]):
                bad.append((seed, i, t))

    ts = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    assert not bad, bad[:5]


def test_resident_container_follows_replacement(pkg):
    """The cached device copy is rebuilt when the directory or a blob is replaced."""
    g = golden_json("decode_d_b5_mem.json")
    c = pkg.CsvContainer.from_bytes(golden_bytes("d_b5_mem"))
    i = int(list(g["bricks"])[1])
    assert h16(c.decode_brick(i, 0)) == g["bricks"][str(i)]["0"][1]
    d = c.directory.copy()
    d[i]["detail_bytes"] = 2          # truncated detail stream: decode must now fail
    c.directory = d
    with pytest.raises(pkg.CorruptStreamError):
        c.decode_brick(i, 0)
    c2 = pkg.CsvContainer.from_bytes(golden_bytes("d_b5_mem"))
    assert h16(c2.decode_brick(i, 1)) == g["bricks"][str(i)]["1"][1]


def test_config1_full_volume(pkg):
    cfg = golden_json("config1.json")
    with open(GOLDEN + "/config1.csv1", "rb") as f:
        c = pkg.CsvContainer.from_bytes(f.read())
    for t in range(6):
        vol = pkg.decompress_volume(c, t)
        assert h16(vol) == cfg["volume"][str(t)], t


def test_slab_partition_equals_whole(pkg):
    """Whole-bz-layer brick ranges (the multi-GPU shard unit) decode to slabs of the full volume."""
    with open(GOLDEN + "/config1.csv1", "rb") as f:
        c = pkg.CsvContainer.from_bytes(f.read())
    full = pkg.decompress_volume(c, 0)
    gx, gy, gz = c.meta.grid_dims
    parts = []
    for (z0, z1) in [(0, 3), (3, 5), (5, 8)]:
        vol = c.to_device(brick_range=(z0 * gx * gy, z1 * gx * gy))
        parts.append(pkg.decompress_volume_device(vol, 0).cpu().numpy().view(np.uint32))
    assert np.array_equal(np.concatenate(parts, axis=0), full)


def test_z_range_rows(pkg):
    """z rows [z0, z1) of the full volume; z0 must sit on a brick boundary (chains read lower rows)."""
    with open(GOLDEN + "/config1.csv1", "rb") as f:
        c = pkg.CsvContainer.from_bytes(f.read())
    vol = c.to_device()
    for t in (0, 1):
        full = pkg.decompress_volume(c, t)
        side = c.meta.brick_side >> t
        z0, z1 = side, min(2 * side + 5, full.shape[0])
        part = pkg.decompress_volume_device(vol, t, z_range=(z0, z1)).cpu().numpy().view(np.uint32)
        assert np.array_equal(part, full[z0:z1])
        with pytest.raises(RuntimeError, match="brick boundary"):
            pkg.decompress_volume_device(vol, t, z_range=(z0 + 1, z1))


@pytest.mark.parametrize("name", ["a_b3", "d_b5_mem", "e_b4_raw", "f_b2_noise", "i_const", "g_b6", "config1"])
def test_stats_matches_reference(pkg, name):
    """stats() (op histogram from K1 count mode) == the reference's stats() output."""
    import json
    exp = golden_json("stats.json")[name]
    path = GOLDEN + ("/config1.csv1" if name == "config1" else f"/vol_{name}.csv1")
    with open(path, "rb") as f:
        c = pkg.CsvContainer.from_bytes(f.read())
    got = json.loads(json.dumps(pkg.stats(c)))
    assert got == exp


@pytest.mark.parametrize("name", ["d_b5_mem", "e_b4_raw"])
def test_cold_container_stats_and_decode(pkg, name):
    """A container opened with detail_cold=True (detail section left on disk,
    container.py:148-159) gives the same stats() and the same volume at every LOD
    as the hot one: the detail streams are read from the file, not taken as empty."""
    import json
    path = GOLDEN + f"/vol_{name}.csv1"
    cold = pkg.CsvContainer.open(path, detail_cold=True)
    assert cold.detail_blob is None
    assert json.loads(json.dumps(pkg.stats(cold))) == golden_json("stats.json")[name]
    g = golden_json(f"decode_{name}.json")
    for t in range(g["brick_log2"] + 1):
        assert h16(pkg.decompress_volume(cold, t)) == g["volume"][str(t)], t
    assert cold.detail_blob is None          # the caller's container stays cold


def test_device_buffers_validated(pkg):
    """Caller-supplied device buffers of the wrong shape, dtype size, layout or
    device are refused before any kernel could index past them."""
    import torch
    c = pkg.CsvContainer.from_bytes(golden_bytes("d_b5_mem"))
    vol = c.to_device()
    cz, cy, cx = vol.crop(0)
    ok = torch.empty((cz, cy, cx), dtype=torch.int32, device="cuda")
    vol.decode(0, out=ok)
    for bad in (torch.empty((cz - 1, cy, cx), dtype=torch.int32, device="cuda"),
                torch.empty((cz, cy, cx), dtype=torch.int16, device="cuda"),
                torch.empty((cz, cx, cy), dtype=torch.int32, device="cuda").transpose(1, 2),
                torch.empty((cz, cy, cx), dtype=torch.int32)):
        with pytest.raises(ValueError):
            vol.decode(0, out=bad)
    with pytest.raises(ValueError, match="results"):
        vol.decode(0, out=ok, results=torch.empty((1, 4), dtype=torch.int64, device="cuda"))
    n = 4
    bricks = torch.arange(n, dtype=torch.int32, device="cuda")
    lods = torch.zeros(n, dtype=torch.uint8, device="cuda")
    dst = torch.arange(n, dtype=torch.int64, device="cuda") * (1 << 3 * c.meta.brick_log2)
    pool = torch.empty(n << 3 * c.meta.brick_log2, dtype=torch.int32, device="cuda")
    vol.decode_bricks(bricks, lods, dst, pool)
    with pytest.raises(ValueError, match="dst"):
        vol.decode_bricks(bricks, lods, dst.to(torch.int32), pool)
    with pytest.raises(ValueError, match="lods"):
        vol.decode_bricks(bricks, lods[:2], dst, pool)
    vol.close()


def test_stats_errors_match_rans_decode(pkg):
    """Corrupted streams raise rans_decode's messages (rans.py:192-197)."""
    with open(GOLDEN + "/vol_d_b5_mem.csv1", "rb") as f:
        data = bytearray(f.read())
    c = pkg.CsvContainer.from_bytes(bytes(data))
    d = c.directory.copy()
    d[3]["detail_bytes"] -= 3          # truncated detail stream of brick 3
    c.directory = d
    with pytest.raises(pkg.CorruptStreamError, match="entropy stream (truncated at symbol|desynchronized)"):
        pkg.stats(c)


def test_mixed_palette_widths(pkg, oracle):
    """One volume whose bricks need both K2w passes (u8 indices for palettes <= 256
    entries, u16 above; both run in the same decode): raster at every LOD and a
    mixed-LOD Morton batch, bit-exact against the oracle."""
    import torch
    rng = np.random.default_rng(11)
    b = 32
    vol = np.zeros((2 * b, 2 * b, 3 * b), dtype=np.uint32)          # (Z, Y, X): 12 bricks
    zz, yy, xx = np.meshgrid(np.arange(2 * b), np.arange(2 * b), np.arange(3 * b), indexing="ij")
    vol[:] = (xx // 9 + 7 * (yy // 11) + 31 * (zz // 13)).astype(np.uint32)   # smooth: small palettes
    for (bz, by, bx) in [(0, 0, 0), (1, 1, 2), (0, 1, 1), (1, 0, 1)]:      # noise bricks: ~32k labels
        vol[bz * b:(bz + 1) * b, by * b:(by + 1) * b, bx * b:(bx + 1) * b] = rng.integers(
            0, 1 << 31, size=(b, b, b), dtype=np.uint32)
    vol[b:, b:, :b][::2, ::3, ::5] = 5                                    # a brick with ~300 labels
    vol[b:, b:, :b][1::2] = rng.integers(0, 300, size=vol[b:, b:, :b][1::2].shape, dtype=np.uint32)
    oc = oracle.compress_volume(vol, brick_log2=5)
    pal = oc.directory[:, 1]
    assert pal.max() > 256 and pal.min() <= 256
    c = pkg.CsvContainer.from_bytes(oc.to_bytes())
    for t in range(6):
        bad, _, ref = oracle.decompress_volume(oc, t)
        assert bad == -1
        assert np.array_equal(pkg.decompress_volume(c, t), ref), t
    v = c.to_device()
    n = oc.n_bricks
    reqs = [(i, t) for i in range(n) for t in (0, 1, 2)]
    sizes = [8 ** (5 - t) for _, t in reqs]
    dst = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    pool = torch.zeros(int(sum(sizes)), dtype=torch.int32, device="cuda")
    res = v.decode_bricks(torch.tensor([r[0] for r in reqs], dtype=torch.int32, device="cuda"),
                          torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device="cuda"),
                          torch.from_numpy(dst).cuda(), pool)
    pkg.GpuVolume.raise_first(res, len(reqs))
    host = pool.cpu().numpy().view(np.uint32)
    for k, (i, t) in enumerate(reqs):
        _, ref = oracle.container_decode_brick(oc, i, t)
        assert np.array_equal(host[dst[k]: dst[k] + sizes[k]], ref), (i, t)


def test_palette_width_boundaries(pkg, oracle):
    """Bricks whose palettes straddle the u8 pass's limit (<= 253 labels: indices
    0-252, bytes 253-255 mark pending neighbour chains) and the u8/u16 split:
    blocky bricks with exactly P labels each (many neighbour ops, P = 1 .. 300),
    plus 1-voxel membranes, every LOD, raster and Morton, against the oracle."""
    import torch
    b = 32
    zz, yy, xx = np.meshgrid(np.arange(b), np.arange(b), np.arange(b), indexing="ij")

    def brick(s_, P, per):   # blocks of s_^3 voxels over P labels, optional 1-voxel planes of label 0
        lab = ((xx // s_) + 16 * (yy // s_) + 256 * (zz // s_)) * 7919 % P
        return np.where((xx + 2 * yy + zz) % per == 0, 0, lab) if per else lab

    # (block, labels, plane period) -> palette length 250 .. 258 (searched with the oracle encoder)
    specs = [(6, 69, 7), (6, 81, 0), (6, 81, 7), (6, 93, 7), (6, 234, 0), (6, 87, 0), (6, 87, 7), (5, 60, 11),
             (6, 159, 7), (4, 9, 0), (8, 3, 5), (6, 40, 7)]
    vol = np.zeros((b, 2 * b, 6 * b), dtype=np.uint32)                  # (Z, Y, X): 12 bricks
    for k, sp in enumerate(specs):
        by, bx = divmod(k, 6)
        vol[:, by * b:(by + 1) * b, bx * b:(bx + 1) * b] = brick(*sp) + 1000 * k
    oc = oracle.compress_volume(vol, brick_log2=5)
    pal = sorted(set(int(v) for v in oc.directory[:, 1]))
    assert set(range(250, 259)) <= set(pal), pal
    c = pkg.CsvContainer.from_bytes(oc.to_bytes())
    for t in range(6):
        bad, _, ref = oracle.decompress_volume(oc, t)
        assert bad == -1
        assert np.array_equal(pkg.decompress_volume(c, t), ref), t
    v = c.to_device()
    n = oc.n_bricks
    reqs = [(i, t) for i in range(n) for t in (0, 1, 2, 3)]
    sizes = [8 ** (5 - t) for _, t in reqs]
    dst = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    pool = torch.zeros(int(sum(sizes)), dtype=torch.int32, device="cuda")
    res = v.decode_bricks(torch.tensor([r[0] for r in reqs], dtype=torch.int32, device="cuda"),
                          torch.tensor([r[1] for r in reqs], dtype=torch.uint8, device="cuda"),
                          torch.from_numpy(dst).cuda(), pool)
    pkg.GpuVolume.raise_first(res, len(reqs))
    host = pool.cpu().numpy().view(np.uint32)
    for k, (i, t) in enumerate(reqs):
        _, ref = oracle.container_decode_brick(oc, i, t)
        assert np.array_equal(host[dst[k]: dst[k] + sizes[k]], ref), (i, t)


def test_cta_fallback_kernel(tmp_path):
    """The CTA-per-brick replay (k2_fast) still serves palettes > 65535 entries; force it
    for a whole process (CSVGPU_K2=cta) and check goldens at every LOD, raster and Morton."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, json, hashlib, numpy as np, torch
sys.path.insert(0, %r)
import paper_2308_16619_b200 as p
from conftest import golden_bytes, golden_json, h16
for name in ["a_b3", "d_b5_mem", "h_b3_u16", "f_b2_noise"]:
    g = golden_json("decode_%%s.json" %% name)
    c = p.CsvContainer.from_bytes(golden_bytes(name))
    for t in range(g["brick_log2"] + 1):
        assert h16(p.decompress_volume(c, t)) == g["volume"][str(t)], (name, t)
print("cta ok")
""" % (os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."),)
    env = dict(os.environ, CSVGPU_K2="cta", PYTHONPATH=os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "cta ok" in r.stdout, r.stderr[-2000:]


def test_k2w6_and_cta_replay_agree(pkg, tmp_path):
    """64^3 replays (b = 64 at LOD 0, b = 128 at LOD 1) run on K2w<6> by default; the
    CTA global-workspace replay (k2_replay<6>) is forced with CSVGPU_K2W6=0 in a
    subprocess.  Both must reproduce the reference goldens at every LOD, raster and
    Morton (the batched test covers Morton through the default path)."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2308_16619_b200 as p
from conftest import golden_bytes, golden_json, h16
for name in ["g_b6", "j_b7"]:
    g = golden_json("decode_%%s.json" %% name)
    c = p.CsvContainer.from_bytes(golden_bytes(name))
    for t in range(g["brick_log2"] + 1):
        assert h16(p.decompress_volume(c, t)) == g["volume"][str(t)], (name, t)
print("k2w6 ok")
""" % (os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."),)
    for flag in ("1", "0"):
        env = dict(os.environ, CSVGPU_K2W6=flag, PYTHONPATH=os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "k2w6 ok" in r.stdout, (flag, r.stderr[-2000:])


def test_side_stream_and_context_manager(pkg):
    """Decodes issued on a non-default stream allocate, launch and check on that stream;
    GpuVolume releases its device memory on leaving a `with` block."""
    import torch
    with open(GOLDEN + "/config1.csv1", "rb") as f:
        c = pkg.CsvContainer.from_bytes(f.read())
    ref = pkg.decompress_volume(c, 0)
    side = torch.cuda.Stream()
    with c.to_device() as vol:
        for t in (0, 1):
            out = pkg.decompress_volume_device(vol, t, stream=side)
            side.synchronize()
            assert np.array_equal(out.cpu().numpy().view(np.uint32), pkg.decompress_volume(c, t))
        n = 64
        bricks = torch.arange(n, dtype=torch.int32, device="cuda")
        lods = torch.zeros(n, dtype=torch.uint8, device="cuda")
        dst = torch.arange(n, dtype=torch.int64, device="cuda") * 32 ** 3
        pool = torch.empty(n * 32 ** 3, dtype=torch.int32, device="cuda")
        res = vol.decode_bricks(bricks, lods, dst, pool, stream=side)
        with torch.cuda.stream(side):
            pkg.GpuVolume.raise_first(res, n)
        side.synchronize()
        pool2 = torch.empty_like(pool)
        pkg.GpuVolume.raise_first(vol.decode_bricks(bricks, lods, dst, pool2), n)
        assert torch.equal(pool, pool2) and ref.size > 0
    assert vol._h is None
