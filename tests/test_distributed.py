"""Multi-rank host logic on CPU (gloo, world sizes 2 and 3): bz-layer sharding,
slab placement and the slab gather of paper_2308_16619_b200.distributed, with
the CPU oracle standing in for the per-rank GPU slab decode."""
import os
import socket

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
    c = orc.Container.from_bytes(container.to_bytes())
    bad, _, vol = orc.decompress_volume(c, t, threads=2, brick_begin=brick_range[0], brick_end=brick_range[1],
                                        z_range=z_range)
    assert bad == -1
    return torch.from_numpy(vol.view(np.int32).copy())


def _worker(rank, world, port, path, t, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    import paper_2308_16619_b200 as p
    from paper_2308_16619_b200.distributed import decompress_volume_distributed
    with open(path, "rb") as f:
        c = p.CsvContainer.from_bytes(f.read())
    full = decompress_volume_distributed(c, t, decode_slab=_oracle_slab)
    if rank == 0:
        q.put(full.numpy().view(np.uint32).copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name,t", [(2, "config1.csv1", 0), (3, "config1.csv1", 1), (3, "vol_d_b5_mem.csv1", 0),
                                           (2, "vol_a_b3.csv1", 2)])
def test_gloo_slab_gather_equals_full_decode(world, name, t):
    from oracle import oracle as orc
    orc.build()
    path = os.path.join(GOLDEN, name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, path, t, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    with open(path, "rb") as f:
        c = orc.Container.from_bytes(f.read())
    bad, _, ref = orc.decompress_volume(c, t)
    assert bad == -1 and np.array_equal(got, ref)


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
