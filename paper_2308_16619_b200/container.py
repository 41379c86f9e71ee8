"""CSV1 container and the whole-volume decode entry points (csvol/container.py).

The on-disk layout (container.py:3-18) is unchanged, so files are
interchangeable with the reference: 32-byte header, two 16 x u16 count
tables, three u64 blob sizes, 44-byte directory rows, palette blob (u32),
coarse blob, detail blob last.

`decompress_volume` keeps the reference signature and return value (a
(Z, Y, X) uint32 numpy volume cropped to ceil(dims / 2^t)); the work runs on
the GPU (K1 entropy lanes + K2/K3 replay-and-raster kernels).
`decompress_volume_device` is the device-resident variant used by the
benchmark: compressed input already in HBM, output left in HBM.
"""

from __future__ import annotations

import dataclasses
import io
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .codec import DIRECTORY_DTYPE, BrickEncoding, decode_brick_entropy, unpack_nibbles
from . import codec
from .errors import ConfigError, CorruptStreamError
from .morton import BrickConfig
from .rans import FrequencyTable, TablePair

MAGIC = b"CSV1"
VERSION = 1
_HEADER = struct.Struct("<4sHBBHH3III")
_BLOBS = struct.Struct("<3Q")
HEAD_LEN = _HEADER.size + 64 + _BLOBS.size


@dataclass(frozen=True)
class VolumeMeta:
    """Shape and encoding parameters (container.py:67-108)."""

    dims: tuple[int, int, int]   # (x, y, z)
    width: int
    brick_log2: int
    entropy: bool = True
    padding_mode: int = 0
    prepass_stride: int = 512

    @property
    def brick_side(self) -> int:
        return 1 << self.brick_log2

    @property
    def grid_dims(self) -> tuple[int, int, int]:
        b = self.brick_side
        return tuple(-(-d // b) for d in self.dims)

    @property
    def padded_dims(self) -> tuple[int, int, int]:
        b = self.brick_side
        return tuple(-(-d // b) * b for d in self.dims)

    @property
    def brick_count(self) -> int:
        gx, gy, gz = self.grid_dims
        return gx * gy * gz

    @property
    def original_bytes(self) -> int:
        x, y, z = self.dims
        return x * y * z * (self.width // 8)

    def brick_index(self, bx: int, by: int, bz: int) -> int:
        gx, gy, _ = self.grid_dims
        return (bz * gy + by) * gx + bx

    def brick_coords(self, index: int) -> tuple[int, int, int]:
        gx, gy, _ = self.grid_dims
        return index % gx, (index // gx) % gy, index // (gx * gy)


@dataclass
class CompressionConfig:
    brick_log2: int = 5
    workers: int | None = None
    prepass_stride: int = 512
    entropy: bool = True


@dataclass
class CsvContainer:
    """A compressed volume in host memory (container.py:119-286)."""

    meta: VolumeMeta
    tables: TablePair
    directory: np.ndarray
    palette_blob: np.ndarray
    coarse_blob: np.ndarray
    detail_blob: np.ndarray | None
    _detail_file: Path | None = field(default=None, repr=False)
    _detail_base: int = field(default=0, repr=False)
    _gpu: object = field(default=None, repr=False, init=False, compare=False)   # (key, GpuVolume) of _device_volume

    @property
    def config(self) -> BrickConfig:
        return BrickConfig(self.meta.brick_log2)

    # -- per-brick accessors -------------------------------------------------
    def brick_palette(self, index: int) -> np.ndarray:
        e = self.directory[index]
        off = int(e["palette_off"])
        return self.palette_blob[off: off + int(e["palette_len"])]

    def brick_coarse(self, index: int) -> np.ndarray:
        e = self.directory[index]
        off = int(e["coarse_off"])
        return self.coarse_blob[off: off + int(e["coarse_bytes"])]

    def brick_detail(self, index: int) -> np.ndarray:
        e = self.directory[index]
        n = int(e["detail_bytes"])
        if self.detail_blob is not None:
            off = int(e["detail_off"])
            return self.detail_blob[off: off + n]
        with open(self._detail_file, "rb") as f:
            f.seek(self._detail_base + int(e["detail_off"]))
            data = f.read(n)
        if len(data) != n:
            raise CorruptStreamError(f"detail section truncated for brick {index}")
        return np.frombuffer(data, dtype=np.uint8)

    def with_detail_loaded(self) -> "CsvContainer":
        """This container with its detail section in memory: ``self`` when it already
        is, else a copy whose detail blob is read from the file of a cold open
        (the bytes brick_detail() would read brick by brick, container.py:148-159)."""
        if self.detail_blob is not None:
            return self
        size = int((self.directory["detail_off"].astype(np.int64) + self.directory["detail_bytes"]).max()) \
            if self.directory.size else 0
        with open(self._detail_file, "rb") as f:
            f.seek(self._detail_base)
            data = f.read(size)
        if len(data) != size:
            raise CorruptStreamError("detail section truncated")
        return dataclasses.replace(self, detail_blob=np.frombuffer(data, dtype=np.uint8).copy())

    def detail_size(self, index: int) -> int:
        return int(self.directory[index]["detail_bytes"])

    def root_labels(self) -> np.ndarray:
        return self.palette_blob[self.directory["palette_off"].astype(np.int64)]

    def decode_brick(self, index: int, t: int, detail: np.ndarray | None = None) -> np.ndarray:
        """Morton-ordered level-t labels of one brick (container.py:168-208), decoded on the GPU."""
        e = self.directory[index]
        cfg = self.config
        if t >= cfg.brick_log2:
            lab = self.brick_palette(index)[:1].astype(np.uint32)
            if t > cfg.brick_log2:
                raise ValueError(f"LOD {t} above coarsest level {cfg.brick_log2}")
            return lab
        if detail is None and (t > 0 or self.detail_blob is not None):
            return self._decode_resident(index, t)
        if t == 0:
            if detail is None:
                detail = self.brick_detail(index)
            n_detail = int(e["detail_nibbles"])
        else:
            detail = np.empty(0, dtype=np.uint8)
            n_detail = 0
        coarse = self.brick_coarse(index)
        if self.meta.entropy:
            return decode_brick_entropy(self.brick_palette(index), coarse, int(e["coarse_nibbles"]), detail,
                                        n_detail, self.tables, t, cfg)
        enc = BrickEncoding(cfg.brick_log2, self.brick_palette(index),
                            unpack_nibbles(coarse, int(e["coarse_nibbles"])), unpack_nibbles(detail, n_detail))
        return codec.decode_brick(enc, t, cfg)

    def _device_volume(self):
        """The container resident in HBM (uploaded on first use, reused by every
        decode_brick call; re-uploaded if the directory or a blob is replaced)."""
        key = (id(self.directory), id(self.palette_blob), id(self.coarse_blob), id(self.detail_blob))
        if self._gpu is None or self._gpu[0] != key:
            if self._gpu is not None:
                self._gpu[1].close()
            self._gpu = (key, self.to_device())
        return self._gpu[1]

    def _decode_resident(self, index: int, t: int) -> np.ndarray:
        """One brick from the device-resident container: one C-ABI call
        (csv_decode_bricks_host: pinned request copy, K1 + K2w, label copy-back)."""
        from . import _lib
        from .device import status_error
        vol = self._device_volume()
        torch = vol._torch
        out = np.empty(8 ** (self.meta.brick_log2 - t), dtype=np.uint32)
        res = np.zeros(1, dtype=_lib.RESULT_DTYPE)
        req_b = np.array([index], dtype=np.uint32)
        req_l = np.array([t], dtype=np.uint8)
        # the C-ABI selects the volume's device itself (cudaSetDevice); the stream is the caller's current one
        _lib.check(_lib.lib().csv_decode_bricks_host(vol._h, 1, req_b.ctypes.data, req_l.ctypes.data,
                                                      out.ctypes.data, res.ctypes.data,
                                                      torch.cuda.current_stream(vol.device).cuda_stream))
        if res["status"][0] != 0:
            raise status_error(int(res["status"][0]), int(res["stream"][0]), int(res["pos"][0]))
        return out

    # -- sizes -----------------------------------------------------------------
    @property
    def payload_bytes(self) -> int:
        return self.palette_blob.size * 4 + self.coarse_blob.size + int(self.directory["detail_bytes"].sum())

    @property
    def compression_rate(self) -> float:
        return self.payload_bytes / self.meta.original_bytes

    # -- serialization -----------------------------------------------------------
    def head_bytes(self) -> bytes:
        """The 120-byte head (header + count tables + blob sizes), container.py:235-253."""
        m = self.meta
        out = _HEADER.pack(MAGIC, VERSION, 1 if m.entropy else 0, m.padding_mode, m.width, m.brick_log2,
                           *m.dims, m.prepass_stride, 0)
        out += self.tables.interior.counts.astype("<u2").tobytes() + self.tables.leaf.counts.astype("<u2").tobytes()
        out += _BLOBS.pack(self.palette_blob.size * 4, self.coarse_blob.size, int(self.directory["detail_bytes"].sum()))
        return out

    def _write_head(self, out) -> None:
        out.write(self.head_bytes())
        out.write(self.directory.astype(DIRECTORY_DTYPE, copy=False).tobytes())
        out.write(self.palette_blob.astype("<u4", copy=False).tobytes())
        out.write(self.coarse_blob.tobytes())

    def to_bytes(self) -> bytes:
        if self.detail_blob is None:
            raise ConfigError("cannot serialize a container with a cold detail section")
        out = io.BytesIO()
        self._write_head(out)
        out.write(self.detail_blob.tobytes())
        return out.getvalue()

    def save(self, path) -> None:
        if self.detail_blob is None:
            raise ConfigError("cannot re-save a container with a cold detail section")
        with open(path, "wb") as f:
            self._write_head(f)
            f.write(self.detail_blob.tobytes())

    @classmethod
    def from_bytes(cls, data: bytes) -> "CsvContainer":
        return _parse(memoryview(data))

    @classmethod
    def open(cls, path, detail_cold: bool = False) -> "CsvContainer":
        path = Path(path)
        if not detail_cold:
            return _parse(memoryview(path.read_bytes()))
        with open(path, "rb") as f:
            head = f.read(HEAD_LEN)
            meta, tables, sizes = _parse_head(head)
            dir_bytes = meta.brick_count * DIRECTORY_DTYPE.itemsize
            rest = f.read(dir_bytes + sizes[0] + sizes[1])
        c = _parse_body(meta, tables, sizes, memoryview(rest))
        c._detail_file = path
        c._detail_base = HEAD_LEN + dir_bytes + sizes[0] + sizes[1]
        return c

    # -- device residency --------------------------------------------------------
    def to_device(self, device=None, brick_range: tuple[int, int] | None = None, cold_detail: bool = False):
        """Upload (a whole-bz-layer brick range of) this container: a GpuVolume.

        With ``cold_detail`` (or when the detail section stayed on disk,
        ``open(..., detail_cold=True)``) the detail blob is not uploaded; level-0
        decodes then read streams staged per frame by a DeviceDetailStream.
        """
        from .device import GpuVolume
        cold_detail = cold_detail or self.detail_blob is None
        b0, b1 = brick_range if brick_range is not None else (0, self.meta.brick_count)
        d = self.directory[b0:b1]
        if b1 > b0:
            p0 = int(d["palette_off"].min())
            p1 = int((d["palette_off"].astype(np.int64) + d["palette_len"]).max())
            c0 = int(d["coarse_off"].min())
            c1 = int((d["coarse_off"].astype(np.int64) + d["coarse_bytes"]).max())
            d0 = int(d["detail_off"].min())
            d1 = int((d["detail_off"].astype(np.int64) + d["detail_bytes"]).max())
        else:
            p0 = p1 = c0 = c1 = d0 = d1 = 0
        p1, c1 = min(p1, self.palette_blob.size), min(c1, self.coarse_blob.size)
        det = np.zeros(0, np.uint8) if cold_detail else self.detail_blob[d0:max(d0, min(d1, self.detail_blob.size))]
        return GpuVolume(self.head_bytes(), d, self.palette_blob[p0:max(p0, p1)], self.coarse_blob[c0:max(c0, c1)],
                         det, brick_begin=b0, brick_end=b1, palette_base=p0,
                         coarse_base=c0, detail_base=d0, device=device)


def _parse_head(head: bytes):
    if len(head) < HEAD_LEN:
        raise CorruptStreamError("container header truncated")
    (magic, version, flags, pad_mode, width, brick_log2, dx, dy, dz, stride, _r) = _HEADER.unpack_from(head, 0)
    if magic != MAGIC:
        raise CorruptStreamError(f"bad magic {magic!r}")
    if version != VERSION:
        raise CorruptStreamError(f"unsupported container version {version}")
    off = _HEADER.size
    interior = np.frombuffer(head, dtype="<u2", count=16, offset=off).astype(np.uint16)
    leaf = np.frombuffer(head, dtype="<u2", count=16, offset=off + 32).astype(np.uint16)
    sizes = _BLOBS.unpack_from(head, off + 64)
    meta = VolumeMeta((dx, dy, dz), width, brick_log2, bool(flags & 1), pad_mode, stride)
    tables = TablePair(FrequencyTable(interior), FrequencyTable(leaf))
    return meta, tables, sizes


def _parse_body(meta, tables, sizes, body: memoryview, detail=None):
    n = meta.brick_count
    dir_bytes = n * DIRECTORY_DTYPE.itemsize
    if len(body) < dir_bytes + sizes[0] + sizes[1]:
        raise CorruptStreamError("container body truncated")
    directory = np.frombuffer(body, dtype=DIRECTORY_DTYPE, count=n)
    off = dir_bytes
    palette = np.frombuffer(body, dtype="<u4", count=sizes[0] // 4, offset=off).astype(np.uint32)
    off += sizes[0]
    coarse = np.frombuffer(body, dtype=np.uint8, count=sizes[1], offset=off).copy()
    return CsvContainer(meta, tables, directory.copy(), palette, coarse, detail)


def _parse(data: memoryview) -> CsvContainer:
    meta, tables, sizes = _parse_head(bytes(data[:HEAD_LEN]))
    body_len = meta.brick_count * DIRECTORY_DTYPE.itemsize + sizes[0] + sizes[1]
    c = _parse_body(meta, tables, sizes, data[HEAD_LEN: HEAD_LEN + body_len])
    detail_off = HEAD_LEN + body_len
    if len(data) < detail_off + sizes[2]:
        raise CorruptStreamError("container detail section truncated")
    c.detail_blob = np.frombuffer(data, dtype=np.uint8, count=sizes[2], offset=detail_off).copy()
    return c


# ------------------------------------------------------------------------------ decode entry points
def _check_t(meta: VolumeMeta, t: int) -> None:
    if not 0 <= t <= meta.brick_log2:
        raise ValueError(f"LOD {t} outside [0, {meta.brick_log2}]")


def decompress_volume_device(container, t: int = 0, out=None, z_range=None, stream=None, check: bool = True):
    """Decode the whole volume at LOD t into a CUDA tensor (int32 storage of u32 labels).

    ``container`` is a CsvContainer (uploaded on the fly) or a GpuVolume
    already resident in HBM.  With ``check`` the lowest failing brick raises
    the reference's CorruptStreamError.
    """
    from .device import GpuVolume, _on_stream
    vol = container if isinstance(container, GpuVolume) else container.to_device()
    if not 0 <= t <= vol.brick_log2:
        raise ValueError(f"LOD {t} outside [0, {vol.brick_log2}]")
    out, res = vol.decode(t, out=out, z_range=z_range, stream=stream)
    if check:
        with _on_stream(vol._torch, vol.device, stream):   # read the results after the decode
            _check_volume_results(vol, t, res)
    return out


def _check_volume_results(vol, t, res):
    """Raise the reference's exception for the lowest failing brick of a volume decode."""
    from .device import GpuVolume
    if t == vol.brick_log2:
        n = vol.n_bricks
        if n and bool((res[:n, 0] & 0xFFFFFFFF).eq(8).any()):
            raise ValueError("expected 1 entries, got shape (0,)")   # morton_to_grid on palette[:1] of an empty palette
    GpuVolume.raise_first(res, vol.n_bricks)


def decompress_volume(container: CsvContainer, t: int = 0, workers: int | None = None, out: np.ndarray | None = None,
                      slab_layers: int | None = None, layers: tuple[int, int] | None = None):
    """Reassemble the volume at LOD t, cropped to ceil(dims / 2**t) (container.py:456-478).

    ``workers`` is accepted for signature compatibility.  The decode runs on the
    GPU in slabs of whole bz layers, double-buffered so that each slab's
    device-to-host copy overlaps the next slab's decode.  ``out`` may be a
    preallocated (ideally pinned) uint32 host array of the cropped shape.
    ``layers=(bz0, bz1)`` decodes only those brick layers (one rank's share of
    a range-partitioned decode, distributed.rank_bricks): the result is that
    z-slab, rows [bz0 * side, min(bz1 * side, cz)), and only its compressed
    bytes are uploaded.
    """
    import torch
    from .device import GpuVolume
    _check_t(container.meta, t)
    meta = container.meta
    x, y, z = meta.dims
    cz, cy, cx = (-(-d // (1 << t)) for d in (z, y, x))
    gx, gy, gz = meta.grid_dims
    side = meta.brick_side >> t
    lz0, lz1 = layers if layers is not None else (0, gz)
    if not 0 <= lz0 <= lz1 <= gz:
        raise ValueError(f"layers {layers} outside [0, {gz}]")
    rz0, rz1 = min(lz0 * side, cz), min(lz1 * side, cz)
    if out is None:
        out = np.empty((rz1 - rz0, cy, cx), dtype=np.uint32)
    elif out.shape != (rz1 - rz0, cy, cx) or out.dtype != np.uint32:
        raise ValueError(f"out must be a uint32 array of shape {(rz1 - rz0, cy, cx)}")
    if container.detail_blob is None:
        if t > 0:   # levels above 0 never read the detail section (container.py:184-190)
            container = dataclasses.replace(container, detail_blob=np.zeros(0, np.uint8))
        else:
            container = container.with_detail_loaded()
    # three-stage pipeline per slab of whole bz layers: upload its compressed
    # bytes (blobs are in brick order, container.py:428-445) -> decode -> D2H
    d = container.directory
    blobs = (container.palette_blob.astype("<u4", copy=False).view(np.uint8), container.coarse_blob,
             container.detail_blob)
    ends = []
    for k, (ocol, lcol, scale) in enumerate((("palette_off", "palette_len", 4), ("coarse_off", "coarse_bytes", 1),
                                              ("detail_off", "detail_bytes", 1))):
        e = (d[ocol].astype(np.int64) + d[lcol].astype(np.int64)) * scale
        ends.append(np.minimum(np.maximum.accumulate(e), blobs[k].size) if e.size else e)
    vol = GpuVolume(container.head_bytes(), d, container.palette_blob.size, container.coarse_blob.size,
                    container.detail_blob.size, deferred=True)
    try:
        n = vol.n_bricks
        dev = vol.device
        nl = lz1 - lz0
        if slab_layers is None:
            slab_layers = max(1, -(-nl // 8))
        layer = gx * gy
        results = torch.empty((max(n, 1), 4), dtype=torch.int64, device=dev)
        host = torch.from_numpy(out.view(np.int32))
        rows = max(1, min(slab_layers * side, rz1 - rz0))
        bufs = [torch.empty((rows, cy, cx), dtype=torch.int32, device=dev) for _ in range(2 if nl > slab_layers else 1)]
        comp = torch.cuda.current_stream(dev)
        up = torch.cuda.Stream(dev)
        # D2H of a slab split over 4 copy streams (one stream reaches ~44-48 GB/s, four ~50);
        # a buffer is reused once all four parts of its previous slab have left it
        copies = [torch.cuda.Stream(dev) for _ in range(4)]
        freed = [[torch.cuda.Event() for _ in copies] for _ in bufs]
        ready = [torch.cuda.Event() for _ in bufs]
        b_first = lz0 * layer
        uploaded = [0, 0, 0]
        if b_first and n:   # a later rank: its blobs start at its first brick's offsets (brick order)
            for k, (ocol, scale) in enumerate((("palette_off", 4), ("coarse_off", 1), ("detail_off", 1))):
                uploaded[k] = min(int(d[ocol][b_first:min(lz1 * layer, n)].min()) * scale, blobs[k].size) \
                    if lz1 > lz0 else 0
        slabs = list(range(lz0, lz1, slab_layers))

        def upload_until(bz1):
            last = min(bz1 * layer, n) - 1
            for k in range(3):
                hi = int(ends[k][last]) if last >= 0 else 0
                if hi > uploaded[k]:
                    vol.upload(k, blobs[k][uploaded[k]:hi], uploaded[k], stream=up)
                    uploaded[k] = hi
            ev = torch.cuda.Event()
            ev.record(up)
            return ev

        up_ev = upload_until(min(lz0 + slab_layers, lz1))
        for k, bz0 in enumerate(slabs):
            bz1 = min(bz0 + slab_layers, lz1)
            z0, z1 = min(bz0 * side, cz), min(bz1 * side, cz)
            i = k % len(bufs)
            comp.wait_event(up_ev)
            if k >= len(bufs):
                for fe in freed[i]:
                    comp.wait_event(fe)
            vol.decode_range(t, bz0 * layer, bz1 * layer, bufs[i], (z0, z1), results[bz0 * layer:], stream=comp)
            ready[i].record(comp)
            nz, nparts = z1 - z0, len(copies)
            for h, cs in enumerate(copies):
                a, b = z0 + nz * h // nparts, z0 + nz * (h + 1) // nparts
                if b > a:
                    cs.wait_event(ready[i])
                    with torch.cuda.stream(cs):
                        host[a - rz0:b - rz0].copy_(bufs[i][a - z0: b - z0], non_blocking=True)
                freed[i][h].record(cs)
            if k + 1 < len(slabs):
                up_ev = upload_until(min(slabs[k + 1] + slab_layers, lz1))
        for s_ in copies:
            s_.synchronize()
        torch.cuda.synchronize(dev)
        lo, hi = b_first, min(lz1 * layer, n)
        res = results[lo:max(hi, lo)]
        if t == meta.brick_log2 and hi > lo and bool((res[:, 0] & 0xFFFFFFFF).eq(8).any()):
            raise ValueError("expected 1 entries, got shape (0,)")   # morton_to_grid on an empty palette[:1]
        GpuVolume.raise_first(res, hi - lo)
    finally:
        vol.close()
    return out


# ------------------------------------------------------------------------------ statistics
_OP_NAMES = ("parent", "neighbor_x", "neighbor_y", "neighbor_z", "palette_last", "palette_back", "palette_advance")


def stats(container: CsvContainer) -> dict:
    """Volume statistics (container.py:498-555): the operation histogram comes
    from the K1 entropy lanes in count mode (csv_volume_op_counts), the per-brick
    rates and palette duplicates from the directory on the host."""
    from .device import GpuVolume   # noqa: F401
    from . import _lib
    meta = container.meta
    d = container.directory
    n = meta.brick_count
    cn = d["coarse_nibbles"].astype(np.int64)
    dn = d["detail_nibbles"].astype(np.int64)
    vol = container.with_detail_loaded().to_device()   # count mode reads every stream, detail included
    try:
        counts, sres = vol.op_counts()
    finally:
        vol.close()
    if meta.entropy:
        # first failing stream in the reference's order: brick by brick, coarse then detail (rans.py:183-198)
        fl = sres["flags"].reshape(n, 2)
        fn = sres["fail_nibble"].reshape(n, 2)
        nn = np.stack([cn, dn], axis=1)
        trunc = (nn > 0) & ((fl & 1) != 0) & ((fl & 8) == 0)
        desync = (nn > 0) & ((fl & 4) != 0)
        bad = trunc | desync
        if bad.any():
            k = int(np.flatnonzero(bad.reshape(-1))[0])
            i, s = divmod(k, 2)
            if trunc[i, s]:
                raise CorruptStreamError(f"entropy stream truncated at symbol {int(fn[i, s])}")
            raise CorruptStreamError(f"entropy stream desynchronized after {int(nn[i, s])} symbols")
    op_counts = counts.astype(np.int64)
    brick_bytes_orig = meta.brick_side ** 3 * (meta.width // 8)
    payload = d["palette_len"].astype(np.int64) * 4 + d["coarse_bytes"].astype(np.int64) + d["detail_bytes"].astype(np.int64)
    brick_cr = payload / brick_bytes_orig
    # palette slices exactly as brick_palette() takes them (numpy slice clamping)
    off = d["palette_off"].astype(np.int64)
    lens = np.clip(np.minimum(off + d["palette_len"].astype(np.int64), container.palette_blob.size) - off, 0, None)
    lens = np.where(off < container.palette_blob.size, lens, 0)
    tot = int(lens.sum())
    if tot:
        starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
        idx = np.arange(tot) - np.repeat(starts - off, lens)
        vals = container.palette_blob[idx]
        bid = np.repeat(np.arange(n), lens)
        order = np.lexsort((vals, bid))
        vs, bs = vals[order], bid[order]
        new = np.ones(tot, dtype=bool)
        new[1:] = (vs[1:] != vs[:-1]) | (bs[1:] != bs[:-1])
        uniq = np.bincount(bs[new], minlength=n)
    else:
        uniq = np.zeros(n, dtype=np.int64)
    duplicates = lens - uniq
    homogeneous = int(((lens == 1) & (cn == 0) & (dn == 0)).sum())
    total_ops = max(int(op_counts.sum()), 1)
    frequencies = {_OP_NAMES[op]: int(op_counts[op]) / total_ops for op in range(7)}
    reuse = sum(frequencies[_OP_NAMES[op]] for op in range(4))
    edges = np.array([0.0] + [2.0 ** e for e in range(-14, 1)])
    hist, _ = np.histogram(brick_cr, bins=edges)
    dup_vals, dup_counts = np.unique(duplicates, return_counts=True)
    return {
        "dims": meta.dims,
        "brick_side": meta.brick_side,
        "brick_count": meta.brick_count,
        "entropy": meta.entropy,
        "original_bytes": meta.original_bytes,
        "payload_bytes": container.payload_bytes,
        "compression_rate": container.compression_rate,
        "op_frequencies": frequencies,
        "reuse_fraction": reuse,
        "total_ops": total_ops,
        "brick_cr_histogram": {"edges": edges.tolist(), "counts": hist.tolist()},
        "brick_cr_max": float(brick_cr.max()) if brick_cr.size else 0.0,
        "homogeneous_bricks": homogeneous,
        "palette_duplicates": dict(zip(dup_vals.tolist(), dup_counts.tolist())),
        "mean_palette_duplicates": float(duplicates.mean()) if duplicates.size else 0.0,
    }
