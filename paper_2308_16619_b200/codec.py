"""Brick codec API: palette + coarse/detail operation streams (csvol/codec.py).

Opcode table (codec.py:9-20, :49-65): each child entry is a nibble
``(stop << 3) | op``; op 5 (palette back-reference) is followed by a payload
nibble delta.  Decoding here runs on the GPU: every function below builds a
one-brick device volume and calls the batched K1/K2 kernels through the
C-ABI, returning Morton-ordered labels exactly as the reference does.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import CorruptStreamError
from .morton import BrickConfig
from .rans import FrequencyTable, TablePair

OP_PARENT = 0
OP_NEIGHBOR_X = 1
OP_NEIGHBOR_Y = 2
OP_NEIGHBOR_Z = 3
OP_PALETTE_LAST = 4
OP_PALETTE_DELTA = 5
OP_PALETTE_ADVANCE = 6

OP_NAMES = {
    OP_PARENT: "parent",
    OP_NEIGHBOR_X: "neighbor_x",
    OP_NEIGHBOR_Y: "neighbor_y",
    OP_NEIGHBOR_Z: "neighbor_z",
    OP_PALETTE_LAST: "palette_last",
    OP_PALETTE_DELTA: "palette_back",
    OP_PALETTE_ADVANCE: "palette_advance",
}

_HEADER = struct.Struct("<4sHBBHH3III")
_BLOBS = struct.Struct("<3Q")
DIRECTORY_DTYPE = np.dtype([
    ("palette_off", "<u8"), ("palette_len", "<u4"),
    ("coarse_off", "<u8"), ("coarse_bytes", "<u4"), ("coarse_nibbles", "<u4"),
    ("detail_off", "<u8"), ("detail_bytes", "<u4"), ("detail_nibbles", "<u4"),
])


@dataclass(frozen=True)
class BrickEncoding:
    """Palette and raw (pre-entropy) nibble streams of one brick (codec.py:70-90)."""

    brick_log2: int
    palette: np.ndarray
    coarse: np.ndarray
    detail: np.ndarray

    @property
    def config(self) -> BrickConfig:
        return BrickConfig(self.brick_log2)

    def __eq__(self, other) -> bool:
        return (isinstance(other, BrickEncoding) and self.brick_log2 == other.brick_log2
                and np.array_equal(self.palette, other.palette) and np.array_equal(self.coarse, other.coarse)
                and np.array_equal(self.detail, other.detail))


def pack_nibbles(nibbles: np.ndarray) -> np.ndarray:
    """Two nibbles per byte, low nibble first (container.py:340-345)."""
    nib = np.asarray(nibbles, dtype=np.uint8)
    if nib.size % 2:
        nib = np.concatenate([nib, np.zeros(1, np.uint8)])
    return (nib[0::2] | (nib[1::2] << 4)).astype(np.uint8)


def unpack_nibbles(packed: np.ndarray, count: int) -> np.ndarray:
    out = np.empty(2 * packed.size, dtype=np.uint8)
    out[0::2] = packed & 0x0F
    out[1::2] = packed >> 4
    return out[:count]


def single_brick_head(brick_log2: int, entropy: bool, tables: TablePair | None,
                      n_pal: int, n_coarse: int, n_detail: int) -> bytes:
    """120-byte CSV1 head of a one-brick volume (layout: container.py:3-18)."""
    b = 1 << brick_log2
    head = _HEADER.pack(b"CSV1", 1, 1 if entropy else 0, 0, 32, brick_log2, b, b, b, 512, 0)
    t = tables or TablePair(FrequencyTable.uniform(), FrequencyTable.uniform())
    head += t.interior.counts.astype("<u2").tobytes() + t.leaf.counts.astype("<u2").tobytes()
    head += _BLOBS.pack(4 * n_pal, n_coarse, n_detail)
    return head


def _decode_one(palette, coarse, n_coarse, detail, n_detail, entropy, tables, config: BrickConfig, t,
                return_consumed):
    """_run_decode (codec.py:498-546) on the GPU for one brick (csv_decode_brick_streams:
    the streams through the library's pinned staging into a cached one-brick volume)."""
    from .device import status_error
    from . import _lib
    palette = np.asarray(palette)
    if palette.size == 0:
        raise CorruptStreamError("empty palette")
    N = config.brick_log2
    if not 0 <= t <= N:
        raise ValueError(f"target LOD {t} outside [0, {N}]")
    if t == N:
        out = palette[:1].astype(np.uint32)
        return (out, 0, 0) if return_consumed else out
    torch = _lib.require_cuda()
    pal = np.ascontiguousarray(palette, dtype=np.uint32)
    cb = np.ascontiguousarray(coarse, dtype=np.uint8)
    db = np.ascontiguousarray(detail, dtype=np.uint8)
    head = single_brick_head(N, entropy, tables, pal.size, cb.size, db.size)
    dev = torch.cuda.current_device()
    out = np.empty(8 ** (N - t), dtype=np.uint32)
    res = np.zeros(1, dtype=_lib.RESULT_DTYPE)
    # one C-ABI call: the library's cached one-brick scratch volume on this device
    _lib.check(_lib.lib().csv_decode_brick_streams(dev, head, pal.ctypes.data, pal.size, cb.ctypes.data, cb.size,
                                                    int(n_coarse), db.ctypes.data, db.size, int(n_detail), t,
                                                    out.ctypes.data, res.ctypes.data,
                                                    torch.cuda.current_stream(dev).cuda_stream))
    r = res[0]
    if r["status"] != 0:
        raise status_error(int(r["status"]), int(r["stream"]), int(r["pos"]))
    if return_consumed:
        return out, int(r["ci"]), int(r["di"])
    return out


def decode_brick(encoding: BrickEncoding, t: int, config: BrickConfig | None = None, return_consumed: bool = False):
    """Raw (pre-entropy) streams -> Morton-ordered level-t labels (codec.py:549-568).

    The nibble arrays are packed two per byte for the device; streams hold
    4-bit symbols (the payload of op 5 is one nibble, SPEC delta in [0, 15]).
    """
    config = config or encoding.config
    c = np.asarray(encoding.coarse, dtype=np.uint8)
    d = np.asarray(encoding.detail, dtype=np.uint8)
    if (c.size and c.max() > 15) or (d.size and d.max() > 15):
        raise ValueError("raw nibble streams must hold 4-bit symbols")
    return _decode_one(encoding.palette, pack_nibbles(c), c.size, pack_nibbles(d), d.size, False, None,
                       config, t, return_consumed)


def decode_brick_entropy(palette, coarse_bytes, coarse_nibbles: int, detail_bytes, detail_nibbles: int,
                         tables: TablePair, t: int, config: BrickConfig, return_consumed: bool = False):
    """Entropy-coded streams -> Morton-ordered level-t labels (codec.py:571-594)."""
    return _decode_one(palette, coarse_bytes, coarse_nibbles, detail_bytes, detail_nibbles, True, tables,
                       config, t, return_consumed)


def encode_brick(pyramid, config: BrickConfig | None = None) -> BrickEncoding:
    """Encode a pyramid into palette + coarse/detail nibble streams (codec.py:224-235).

    Runs the GPU encoder's per-brick stages (csv_encode_volume: E1 pyramid, E2
    greedy operations + palette replay, raw nibble packing) on the brick's
    level-0 labels.  Those stages re-derive levels 1..N, so ``pyramid`` must
    be the reference rule's pyramid of its level 0 (what build_pyramid
    returns); any other pyramid is refused with ValueError rather than encoded
    differently from the reference.
    """
    from .container import CompressionConfig
    from .encode import compress_volume
    from .morton import morton_to_grid
    from .pyramid import build_pyramid
    config = config or pyramid.config
    n = config.brick_log2
    level0 = np.ascontiguousarray(pyramid.levels[0], dtype=np.uint32)
    if level0.shape != (8 ** n,) or len(pyramid.levels) != n + 1:
        raise ValueError(f"pyramid does not match b={config.side}")
    ref = build_pyramid(level0, config)
    if any(not np.array_equal(np.asarray(a), b) for a, b in zip(pyramid.levels, ref.levels)) or \
            any(not np.array_equal(np.asarray(a, dtype=bool), b) for a, b in zip(pyramid.constant, ref.constant)):
        raise ValueError("pyramid is not the mode-of-8 pyramid of its level 0 (build_pyramid)")
    grid = morton_to_grid(level0, config.side)
    c = compress_volume(grid, CompressionConfig(brick_log2=n, entropy=False))
    e = c.directory[0]
    coarse = unpack_nibbles(c.brick_coarse(0), int(e["coarse_nibbles"]))
    detail = unpack_nibbles(c.brick_detail(0), int(e["detail_nibbles"]))
    return BrickEncoding(n, c.brick_palette(0).astype(np.uint32).copy(), coarse.copy(), detail.copy())


def decode_root(encoding: BrickEncoding) -> int:
    """Coarsest-LOD label (codec.py:597-601)."""
    if encoding.palette.size == 0:
        raise CorruptStreamError("empty palette")
    return int(encoding.palette[0])


def iter_operations(nibbles: np.ndarray):
    """(opcode, stop, delta) triples of one raw nibble stream (codec.py:604-623)."""
    i, n = 0, nibbles.size
    while i < n:
        nib = int(nibbles[i])
        i += 1
        op, stop, delta = nib & 7, nib >> 3, None
        if op == OP_PALETTE_DELTA:
            if i >= n:
                raise CorruptStreamError(f"stream underrun (payload nibble {i})")
            delta = int(nibbles[i])
            i += 1
        yield op, stop, delta
