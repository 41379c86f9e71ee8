"""Multi-rank host logic on CPU (gloo, world sizes 2 and 3): bz-layer sharding,
slab placement, the gather-to-root (grouped isend/irecv) and gather-to-all
(all_gather_into_tensor / per-owner broadcast) of
paper_2308_16619_b200.distributed, and the collective error agreement, with the
CPU oracle standing in for the per-rank GPU slab decode.  The bench's strong
scaling driver (bench.strong_rank_plan) is checked against the same partition."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_slab(container, brick_range, z_range, t):
    from oracle import oracle as orc
    from paper_2308_16619_b200.distributed import NO_ERROR
    c = orc.Container.from_bytes(container.to_bytes())
    bad, res, vol = orc.decompress_volume(c, t, threads=2, brick_begin=brick_range[0], brick_end=brick_range[1],
                                          z_range=z_range)
    err = torch.tensor([NO_ERROR if bad < 0 else bad, res[0], res[1], res[2]], dtype=torch.int64)
    return err, torch.from_numpy(vol.view(np.int32).copy())


def _worker(rank, world, port, data, t, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import paper_2308_16619_b200 as p
    from paper_2308_16619_b200.distributed import decompress_volume_distributed
    c = p.CsvContainer.from_bytes(data)
    try:
        got = decompress_volume_distributed(c, t, gather=mode, decode_slab=_oracle_slab)
        q.put((rank, "ok", got.numpy().view(np.uint32).copy()))
    except Exception as e:   # every rank must raise the same exception
        q.put((rank, type(e).__name__, str(e)))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, data, t, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, data, t, mode, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict((r, (k, v)) for r, k, v in (q.get(timeout=300) for _ in range(world)))
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    return out


@pytest.mark.parametrize("world,name,t,mode", [(2, "config1.csv1", 0, "all"), (3, "config1.csv1", 1, "root"),
                                                (3, "vol_d_b5_mem.csv1", 0, "all"), (2, "vol_a_b3.csv1", 2, "root"),
                                                (2, "config1.csv1", 5, "all")])
def test_gloo_slab_gather_equals_full_decode(world, name, t, mode):
    from oracle import oracle as orc
    orc.build()
    with open(os.path.join(GOLDEN, name), "rb") as f:
        data = f.read()
    out = _run(world, data, t, mode)
    c = orc.Container.from_bytes(data)
    bad, _, ref = orc.decompress_volume(c, t)
    assert bad == -1
    from paper_2308_16619_b200.distributed import rank_slab
    for r, (kind, got) in out.items():
        assert kind == "ok", got
        if mode == "all" or r == 0:
            assert np.array_equal(got, ref), f"rank {r}"
        else:   # the root-gather's senders keep their own slab
            z0, z1 = rank_slab(c.dims, c.brick_log2, t, world, r)
            assert np.array_equal(got, ref[z0:z1]), f"rank {r}"


def test_gloo_error_agreement():
    """A corrupt stream in rank 1's bricks: every rank raises the reference's message for the
    globally lowest failing brick (container.py:470-478), nobody hangs in the gather."""
    from oracle import oracle as orc
    orc.build()
    with open(os.path.join(GOLDEN, "config1.csv1"), "rb") as f:
        data = bytearray(f.read())
    c = orc.Container.from_bytes(bytes(data))
    gx, gy, gz = c.grid
    layer = gx * gy
    # corrupt the coarse streams of two bricks of the upper half (rank 1 of 2) and one of rank 2 of 3
    import paper_2308_16619_b200 as p
    pc = p.CsvContainer.from_bytes(bytes(data))
    for b in (5 * layer + 3, 6 * layer + 1, 7 * layer):
        e = pc.directory[b]
        if int(e["coarse_bytes"]) > 6:
            pc.coarse_blob[int(e["coarse_off"]) + 2] ^= 0x5A
            pc.coarse_blob[int(e["coarse_off"]) + 5] ^= 0xC3
    bad_data = pc.to_bytes()
    cb = orc.Container.from_bytes(bad_data)
    bad, res, _ = orc.decompress_volume(cb, 0)
    assert bad >= 0
    want = orc.error_message(res[0], res[1], res[2])
    for world in (2, 3):
        out = _run(world, bad_data, 0, "root")
        for r, (kind, msg) in out.items():
            assert kind == "CorruptStreamError" and msg == want, (r, kind, msg, want)


def test_partition_covers_volume():
    from paper_2308_16619_b200.distributed import bz_range, rank_slab
    for gz in (1, 2, 7, 64):
        for world in (1, 2, 3, 8):
            spans = [bz_range(gz, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == gz
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    dims = (70, 64, 40)
    for t in range(6):
        rows = [rank_slab(dims, 5, t, 3, r) for r in range(3)]
        assert rows[0][0] == 0 and rows[-1][1] == -(-40 // (1 << t))


def test_bench_strong_plan_partitions_one_volume():
    """bench.py --gpus N (strong, the default): the N ranks' brick ranges and slabs tile ONE volume."""
    sys.path.insert(0, ROOT)
    import bench
    for world in (1, 2, 4, 8):
        plans = [bench.strong_rank_plan((2048, 2048, 2048), 5, world, r) for r in range(world)]
        assert plans[0]["bricks"][0] == 0 and plans[-1]["bricks"][1] == 64 ** 3
        assert plans[0]["rows"][0] == 0 and plans[-1]["rows"][1] == 2048
        for a, b in zip(plans, plans[1:]):
            assert a["bricks"][1] == b["bricks"][0] and a["rows"][1] == b["rows"][0]
        assert sum(pl["voxels"] for pl in plans) == 2048 ** 3
