"""Multi-GPU decode: bricks range-partitioned on whole bz layers.

Bricks are independent (no cross-brick references), so rank r
decodes bz layers [bz0, bz1) with no data-path collective: its palette,
coarse and detail data are contiguous blob slices (brick-order blobs,
container.py:428-445) and its output is the contiguous raster z-slab
[bz0*side, min(bz1*side, Z)) x Y x X.  The only exchange is the optional
final gather of the decoded slabs (NCCL all_gather over NVLink).
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def bz_range(gz: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of gz brick layers over `world` ranks."""
    base, extra = divmod(gz, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def rank_bricks(grid: tuple[int, int, int], world: int, rank: int) -> tuple[int, int]:
    """Brick-index range [b0, b1) of this rank's whole bz layers."""
    gx, gy, gz = grid
    z0, z1 = bz_range(gz, world, rank)
    return z0 * gx * gy, z1 * gx * gy


def rank_slab(dims: tuple[int, int, int], brick_log2: int, t: int, world: int, rank: int) -> tuple[int, int]:
    """LOD-t raster z rows [z0, z1) owned by this rank (container.py:476-478 crop)."""
    side = (1 << brick_log2) >> t
    gz = -(-dims[2] // (1 << brick_log2))
    cz = -(-dims[2] // (1 << t))
    b0, b1 = bz_range(gz, world, rank)
    return min(b0 * side, cz), min(b1 * side, cz)


def decompress_volume_distributed(container, t: int = 0, group=None, gather: bool = True,
                                  decode_slab: Callable | None = None):
    """Decode this rank's slab; optionally all-gather the full cropped volume.

    ``decode_slab(container, brick_range, z_range, t) -> (z1-z0, Y, X) tensor``
    defaults to the GPU path (container.to_device + csv_decode_volume).  With
    ``gather`` every rank returns the full volume (slabs exchanged with one
    all_gather of equal-sized, zero-padded slabs); otherwise its own slab.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    meta = container.meta
    grid = meta.grid_dims
    b0, b1 = rank_bricks(grid, world, rank)
    z0, z1 = rank_slab(meta.dims, meta.brick_log2, t, world, rank)
    if decode_slab is None:
        from .container import decompress_volume_device
        vol = container.to_device(brick_range=(b0, b1))
        slab = decompress_volume_device(vol, t, z_range=(z0, z1))
    else:
        slab = decode_slab(container, (b0, b1), (z0, z1), t)
    if not gather or world == 1:
        return slab
    x, y, z = meta.dims
    cz, cy, cx = (-(-d // (1 << t)) for d in (z, y, x))
    rows = max(rank_slab(meta.dims, meta.brick_log2, t, world, r)[1] - rank_slab(meta.dims, meta.brick_log2, t, world, r)[0]
               for r in range(world))
    pad = torch.zeros((rows, cy, cx), dtype=slab.dtype, device=slab.device)
    pad[: slab.shape[0]] = slab
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    parts = []
    for r in range(world):
        s0, s1 = rank_slab(meta.dims, meta.brick_log2, t, world, r)
        parts.append(bufs[r][: s1 - s0])
    return torch.cat(parts, dim=0)
