"""Multi-GPU decode: bricks range-partitioned on whole bz layers.

Bricks are independent (no cross-brick references), so rank r
decodes bz layers [bz0, bz1) with no data-path collective: its palette,
coarse and detail data are contiguous blob slices (brick-order blobs,
container.py:428-445) and its output is the contiguous raster z-slab
[bz0*side, min(bz1*side, Z)) x Y x X.  The reference's thread pool over
bricks (container.py:470-472) becomes this range partition over ranks.

The only data exchange is the final gather of the decoded slabs:

* ``gather="root"``: grouped point-to-point (``batch_isend_irecv`` =
  ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd) straight into the
  root's preallocated (Z, Y, X) volume -- each peer's slab lands in its own
  contiguous z-row view, the root decodes its own slab in place, no padding
  and no concatenation.
* ``gather="peer"`` (fused decode + gather): the root allocates the volume as an
  IPC-shareable buffer (csv_peer_alloc) and broadcasts its 64-byte handle; every
  other rank maps it (csv_peer_open: NVLink peer memory on a multi-GPU node) and
  decodes its slab with the output pointer INSIDE the root's volume, so the K2w
  row stores go straight to the root while the rest of the slab is still being
  decoded -- no NCCL data-path collective, no staging buffer.  The root returns a
  PeerVolume (``.tensor()`` is the volume); the others return None.
* ``gather="all"``: every rank ends with the volume.  Equal slabs (the
  2048^3 / 1024^3 workloads on 1, 2, 4, 8 ranks) use one
  ``all_gather_into_tensor`` into the output itself; unequal ones one
  broadcast per owner into its row view.

Errors: every rank decodes without raising, then the ranks exchange their
lowest failing global brick (status, stream, nibble) so that all ranks raise
the same exception -- the one the reference raises for the lowest failing
brick of the whole volume (container.py:470-478 walks bricks in order) --
and nobody is left blocked in the gather.
"""

from __future__ import annotations

from typing import Callable

import numpy as np

NO_ERROR = np.iinfo(np.int64).max


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


def first_error(results, n: int, brick_begin: int, device=None):
    """(global brick, status, stream, pos) of the lowest failing brick in a results
    table (csv_result rows as int64[n, 4]), or (NO_ERROR, 0, 0, 0)."""
    import torch
    if n:
        st = results[:n, 0] & 0xFFFFFFFF
        bad = st.nonzero()
        if bad.numel():
            i = int(bad[0, 0])
            from . import _lib
            row = results[i].cpu().numpy().view(_lib.RESULT_DTYPE)[0]
            return torch.tensor([brick_begin + i, int(row["status"]), int(row["stream"]), int(row["pos"])],
                                dtype=torch.int64, device=device)
    return torch.tensor([NO_ERROR, 0, 0, 0], dtype=torch.int64, device=device)


def agree_on_error(err, group=None):
    """All-gather every rank's (brick, status, stream, pos) and return the row of the
    globally lowest failing brick (NO_ERROR if none): the same on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return err
    # NCCL exchanges device tensors; gloo (CPU tests, the single-device peer test) host ones
    dev = err.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    allv = torch.empty((world, 4), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allv, err.reshape(1, 4).to(dev).contiguous(), group=group)
    return allv[int(torch.argmin(allv[:, 0]))]


def raise_agreed(err) -> None:
    brick, status, stream, pos = (int(v) for v in err.cpu().tolist())
    if brick == NO_ERROR:
        return
    from .device import status_error
    raise status_error(status, stream, pos)


def gather_slabs(slab, out, dims, brick_log2: int, t: int, mode: str = "root", root: int = 0, group=None):
    """Exchange decoded slabs.  ``slab`` is this rank's (z1-z0, cy, cx) rows (for the
    root / every rank in "all" mode it may already be the view ``out[z0:z1]``);
    ``out`` the (cz, cy, cx) volume on the receiving rank(s), None elsewhere."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    spans = [rank_slab(dims, brick_log2, t, world, r) for r in range(world)]
    z0, z1 = spans[rank]
    if mode == "root":
        if rank == root:
            if slab.data_ptr() != out[z0:z1].data_ptr():
                out[z0:z1].copy_(slab)
            ops = [dist.P2POp(dist.irecv, out[a:b], dist.get_global_rank(group, r) if group is not None else r,
                              group=group)
                   for r, (a, b) in enumerate(spans) if r != root and b > a]
        else:
            ops = [dist.P2POp(dist.isend, slab, dist.get_global_rank(group, root) if group is not None else root,
                              group=group)] if z1 > z0 else []
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return out if rank == root else slab
    if mode != "all":
        raise ValueError(f"gather mode {mode!r} is not 'root' or 'all'")
    if slab.data_ptr() != out[z0:z1].data_ptr():
        out[z0:z1].copy_(slab)
    rows = [b - a for a, b in spans]
    if all(r == rows[0] for r in rows) and rows[0] * world == out.shape[0]:
        # equal slabs: one collective writes every slab straight into place (the local one
        # is its own input, an in-place all-gather)
        dist.all_gather_into_tensor(out, out[z0:z1], group=group)
    else:
        for r, (a, b) in enumerate(spans):
            if b > a:
                dist.broadcast(out[a:b], dist.get_global_rank(group, r) if group is not None else r, group=group)
    return out


class _CudaArray:
    """A raw device pointer seen by torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(int(v) for v in shape), "typestr": "<i4",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class PeerVolume:
    """The root's (cz, cy, cx) int32 volume in IPC-shareable device memory.

    ``PeerVolume.alloc(shape, device)`` on the root (``handle`` = 64 bytes to publish),
    ``PeerVolume.open(handle, shape, device)`` on the other ranks.  ``rows_ptr(z)`` is the
    device address of row z (what a rank passes to the decode); ``tensor()`` views the
    whole volume on the root.  ``close()`` frees (root) or unmaps (others)."""

    def __init__(self, ptr: int, shape, device, handle: bytes, owner: bool):
        self.ptr, self.shape, self.device, self.handle, self.owner = ptr, tuple(shape), device, handle, owner

    @classmethod
    def alloc(cls, shape, device):
        import ctypes
        from . import _lib
        nbytes = 4 * int(np.prod(shape, dtype=np.int64))
        p = ctypes.c_void_p()
        h = (ctypes.c_uint8 * 64)()
        _lib.check(_lib.lib().csv_peer_alloc(device.index, nbytes, ctypes.byref(p), h))
        return cls(p.value, shape, device, bytes(h), True)

    @classmethod
    def open(cls, handle: bytes, shape, device):
        import ctypes
        from . import _lib
        p = ctypes.c_void_p()
        h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
        _lib.check(_lib.lib().csv_peer_open(device.index, h, ctypes.byref(p)))
        return cls(p.value, shape, device, handle, False)

    def rows_ptr(self, z: int) -> int:
        return self.ptr + 4 * int(z) * self.shape[1] * self.shape[2]

    def tensor(self):
        import torch
        t = torch.as_tensor(_CudaArray(self.ptr, self.shape), device=self.device)
        t._peer_volume = self          # keep the allocation alive with the view
        return t

    def close(self) -> None:
        from . import _lib
        if self.ptr:
            (_lib.lib().csv_peer_free if self.owner else _lib.lib().csv_peer_close)(self.device.index, self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decompress_volume_peer(container, t: int = 0, group=None, root: int = 0):
    """Fused decode + gather (``gather="peer"`` above): every rank decodes its
    whole-bz-layer slab straight into the root's volume through peer memory.
    Returns the root's PeerVolume on the root, None elsewhere; raises the
    reference's exception for the globally lowest failing brick on every rank."""
    import torch
    import torch.distributed as dist
    from . import _lib
    torch_ = _lib.require_cuda()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    meta = container.meta
    if not 0 <= t <= meta.brick_log2:
        raise ValueError(f"LOD {t} outside [0, {meta.brick_log2}]")
    x, y, z = meta.dims
    shape = tuple(-(-d // (1 << t)) for d in (z, y, x))
    dev = torch_.device("cuda", torch_.cuda.current_device())
    pv = PeerVolume.alloc(shape, dev) if rank == root else None
    if world > 1:
        box = [pv.handle if pv is not None else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, root) if group is not None else root,
                                   group=group)
        if pv is None:
            pv = PeerVolume.open(box[0], shape, dev)
    b0, b1 = rank_bricks(meta.grid_dims, world, rank)
    z0, z1 = rank_slab(meta.dims, meta.brick_log2, t, world, rank)
    vol = container.to_device(device=dev, brick_range=(b0, b1))
    try:
        res = torch_.empty((max(vol.n_bricks, 1), 4), dtype=torch_.int64, device=dev)
        if z1 > z0:
            vol.decode_into(t, pv.rows_ptr(z0), (z0, z1), res)
        torch_.cuda.current_stream(dev).synchronize()      # this rank's rows have landed in the root's volume
        err = first_error(res, vol.n_bricks, b0, device=dev)
        if t == meta.brick_log2 and vol.n_bricks and bool((res[:vol.n_bricks, 0] & 0xFFFFFFFF).eq(8).any()):
            err = torch_.tensor([b0, -1, 0, 0], dtype=torch_.int64, device=dev)
    finally:
        vol.close()
    err = agree_on_error(err, group)
    if world > 1:
        dist.barrier(group=group)                            # every slab is in place
    if rank != root:
        pv.close()
    try:
        if int(err[1]) == -1:
            raise ValueError("expected 1 entries, got shape (0,)")
        raise_agreed(err)
    except Exception:
        if rank == root:
            pv.close()
        raise
    return pv if rank == root else None


def decompress_volume_distributed(container, t: int = 0, group=None, gather: str | bool | None = "all",
                                  root: int = 0, out=None, decode_slab: Callable | None = None):
    """Decode this rank's whole-bz-layer slab and gather the cropped (Z, Y, X) volume.

    ``container``: a CsvContainer (each rank uploads only its brick range).
    ``gather``: "all" (every rank returns the volume), "root" (rank ``root``
    returns it, the others their slab), None / False (each rank its slab).
    ``out``: optional preallocated (cz, cy, cx) int32 tensor on the receiving
    rank(s); the local slab is decoded straight into its rows.
    ``decode_slab(container, brick_range, z_range, t) -> (err, slab)`` replaces
    the GPU decode (CPU tests; ``err`` = int64[4] (global brick, status,
    stream, pos) of the slab's lowest failing brick, brick NO_ERROR if none);
    by default the slab is decoded by csv_decode_volume and the per-brick
    statuses are checked collectively.
    """
    import torch
    import torch.distributed as dist
    if gather is True:
        gather = "all"
    if gather == "peer":
        pv = decompress_volume_peer(container, t, group=group, root=root)
        return pv.tensor() if pv is not None else None
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    meta = container.meta
    if not 0 <= t <= meta.brick_log2:
        raise ValueError(f"LOD {t} outside [0, {meta.brick_log2}]")
    x, y, z = meta.dims
    cz, cy, cx = (-(-d // (1 << t)) for d in (z, y, x))
    b0, b1 = rank_bricks(meta.grid_dims, world, rank)
    z0, z1 = rank_slab(meta.dims, meta.brick_log2, t, world, rank)
    receives = gather == "all" or (gather == "root" and rank == root) or world == 1
    if decode_slab is None:
        from . import _lib
        _lib.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device())
        if receives and out is None:
            out = torch.empty((cz, cy, cx), dtype=torch.int32, device=dev)
        vol = container.to_device(device=dev, brick_range=(b0, b1))
        try:
            slab, res = vol.decode(t, out=out[z0:z1] if receives else None, z_range=(z0, z1))
            err = first_error(res, vol.n_bricks, b0, device=dev)
            if t == meta.brick_log2 and vol.n_bricks and bool((res[:vol.n_bricks, 0] & 0xFFFFFFFF).eq(8).any()):
                err = torch.tensor([b0, -1, 0, 0], dtype=torch.int64, device=dev)
        finally:
            vol.close()
    else:
        err, slab = decode_slab(container, (b0, b1), (z0, z1), t)
        if receives and out is None:
            out = torch.empty((cz, cy, cx), dtype=slab.dtype, device=slab.device)
        if receives:
            out[z0:z1].copy_(slab)
            slab = out[z0:z1]
    err = agree_on_error(err, group)
    if int(err[1]) == -1:   # morton_to_grid on palette[:1] of an empty palette (coarsest LOD)
        raise ValueError("expected 1 entries, got shape (0,)")
    raise_agreed(err)
    if world == 1:
        return out if receives else slab
    if not gather:
        return slab
    return gather_slabs(slab, out, meta.dims, meta.brick_log2, t, mode=gather, root=root, group=group)
