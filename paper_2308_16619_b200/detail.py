"""Cold-detail streaming for the cache decode.

The reference keeps a container's detail section (the level-0 streams, the
bulk of the bytes) on disk and fetches at most ``budget_bytes`` of requested
streams per frame; bricks whose stream did not fit decode at level 1 this
frame (DetailStore, render.py:782-832; cold reads, container.py:148-159).

`DetailStore` is that planner, unchanged.  `DeviceDetailStream` adds the GPU
side: the streams a frame's level-0 placements need (fetched ones from
``hot``, the rest read synchronously like FrameLoop._decode, render.py:876-885)
are packed into a pinned host buffer, copied to a device staging buffer in one
asynchronous H2D transfer, and pointed at by the volume's directory
(csv_volume_stage_detail) right before the batched decode.  The device volume
itself never holds the detail blob.
"""

from __future__ import annotations

import ctypes
from collections.abc import Sequence

import numpy as np

from . import _lib


class FallbackLog(Sequence):
    """The (frame, brick) fallback list of DetailStore, kept as one brick array per
    frame so a 40k-brick frame costs one array copy; it reads like the reference's
    list of tuples (len, indexing, iteration, ==)."""

    def __init__(self):
        self._chunks: list[tuple[int, np.ndarray]] = []
        self._n = 0
        self._flat = None

    def append(self, item) -> None:
        self._chunks.append((int(item[0]), np.array([item[1]], dtype=np.int64)))
        self._n += 1
        self._flat = None

    def extend_frame(self, frame: int, bricks: np.ndarray) -> None:
        if bricks.size:
            self._chunks.append((int(frame), np.array(bricks, dtype=np.int64)))
            self._n += int(bricks.size)
            self._flat = None

    def clear(self) -> None:
        self._chunks, self._n, self._flat = [], 0, None

    def _list(self) -> list:
        if self._flat is None:
            self._flat = [(f, b) for f, a in self._chunks for b in a.tolist()]
        return self._flat

    def __len__(self) -> int:
        return self._n

    def __getitem__(self, i):
        return self._list()[i]

    def __eq__(self, other) -> bool:
        return self._list() == list(other)

    def __repr__(self) -> str:
        return repr(self._list())


class DetailStore:
    """Budgeted access to the cold detail section of a container (render.py:782-832)."""

    def __init__(self, container, budget_bytes: int = 8 << 20):
        self.container = container
        self.budget_bytes = budget_bytes
        self.hot: dict[int, np.ndarray] = {}
        self.fetched_bytes_total = 0
        self.deferred_last_frame = 0
        self.fallback_log = FallbackLog()  # (frame, brick) pairs
        self._frame = 0

    def plan(self, requests) -> list[tuple[int, int]]:
        """Fetch detail for level-0 requests within budget; downgrade the rest to level 1."""
        if len(requests) > 256:             # same result, vectorised (numpy + the C budget scan)
            b, l = self.plan_arrays(requests)
            return list(zip(b.tolist(), l.tolist()))
        spent = 0
        deferred = 0
        adjusted: list[tuple[int, int]] = []
        for brick, lod in sorted(set(requests)):
            if lod != 0:
                adjusted.append((brick, lod))
                continue
            size = self.container.detail_size(brick)
            if size == 0 or brick in self.hot:
                adjusted.append((brick, 0))
                continue
            if spent + size <= self.budget_bytes:
                self.hot[brick] = self.container.brick_detail(brick)
                spent += size
                self.fetched_bytes_total += size
                adjusted.append((brick, 0))
            else:
                deferred += 1
                self.fallback_log.append((self._frame, brick))
                if self.container.meta.brick_log2 >= 2:
                    adjusted.append((brick, 1))
        self.deferred_last_frame = deferred
        self._frame += 1
        return adjusted

    def plan_arrays(self, requests):
        """plan() with numpy: (bricks int64, lods int64) of the adjusted, sorted, unique requests."""
        r = np.asarray(requests, dtype=np.int64).reshape(-1, 2)
        key = np.sort(r[:, 0] * 256 + r[:, 1])                    # sorted(set(requests))
        if key.size > 1:
            key = key[np.concatenate(([True], key[1:] != key[:-1]))]
        bricks, lods = key >> 8, key & 255
        lod0 = lods == 0
        if getattr(self, "_dir64", None) is None:      # the directory is immutable: convert once
            d = self.container.directory
            self._dir64 = (d["detail_bytes"].astype(np.int64), d["detail_off"].astype(np.int64))
        sizes = self._dir64[0][bricks]
        hot = np.fromiter(self.hot.keys(), dtype=np.int64, count=len(self.hot))
        cand = lod0 & (sizes > 0) & ~np.isin(bricks, hot)
        cs = np.ascontiguousarray(sizes[cand], dtype=np.uint64)
        acc = np.zeros(cs.size, dtype=np.uint8)
        spent = ctypes.c_uint64()
        _lib.check(_lib.lib().csv_detail_plan_greedy(cs.ctypes.data, cs.size, int(self.budget_bytes),
                                                     acc.ctypes.data, ctypes.byref(spent)))
        ci = np.flatnonzero(cand)
        fetched, deferred = ci[acc == 1], ci[acc == 0]
        fb = bricks[fetched]
        blob = getattr(self.container, "detail_blob", None)
        if blob is not None and fb.size:         # in-memory detail: slice views in one pass
            offs = self._dir64[1][fb].tolist()
            lens = self._dir64[0][fb].tolist()
            self.hot.update({b: blob[o: o + n] for b, o, n in zip(fb.tolist(), offs, lens)})
        else:
            for b in fb.tolist():
                self.hot[b] = self.container.brick_detail(b)
        self.fetched_bytes_total += int(sizes[fetched].sum())
        self.deferred_last_frame = int(deferred.size)
        self.fallback_log.extend_frame(self._frame, bricks[deferred])
        self._frame += 1
        keep = np.ones(bricks.size, dtype=bool)
        out_l = lods.copy()
        if self.container.meta.brick_log2 >= 2:
            out_l[deferred] = 1
        else:
            keep[deferred] = False
        return bricks[keep], out_l[keep]

    def take(self, brick: int):
        """Hand the fetched stream to the decoder; it is not kept afterwards."""
        return self.hot.pop(brick, None)


class DeviceDetailStream(DetailStore):
    """DetailStore whose streams reach the GPU decoder through one staged H2D copy per frame."""

    def __init__(self, container, volume, budget_bytes: int = 8 << 20):
        super().__init__(container, budget_bytes)
        self.volume = volume
        torch = volume._torch
        self._torch = torch
        self._cap = 0
        self._host = None
        self._dev = None
        self._dev_stream = None
        self.staged_bytes_total = 0
        self.staged_last_frame = 0
        self._ev = None

    def _ensure(self, nbytes: int, stream):
        """Grow the staging buffers.  The device buffer is allocated on, and its
        predecessor released against, the stream the decodes that read it run
        on (the caller's), so a decode still reading the old buffer keeps it alive."""
        torch = self._torch
        if nbytes > self._cap:
            cap = max(nbytes, 1 << 16)
            self._host = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            if self._dev is not None and self._dev_stream is not None:
                self._dev.record_stream(self._dev_stream)
            with torch.cuda.device(self.volume.device), torch.cuda.stream(stream):
                self._dev = torch.empty(cap + 64, dtype=torch.uint8, device=self.volume.device)
            self._cap = cap
        self._dev_stream = stream

    def stage(self, bricks, stream=None) -> None:
        """Make the level-0 streams of `bricks` readable by the next decode (take semantics)."""
        from .device import _ptr, _stream_handle
        torch = self._torch
        if self._ev is not None:
            self._ev.synchronize()              # the previous frame's copy has left the pinned buffer
        bricks = [int(b) for b in bricks]
        streams = []
        for b in bricks:
            s = self.take(b)
            if s is None:                       # not fetched this frame: read it now (render.py:876-878)
                s = self.container.brick_detail(b)
            streams.append(np.asarray(s, dtype=np.uint8))
        lens = np.array([s.size for s in streams], dtype=np.int64)
        offs = np.zeros(len(streams), dtype=np.int64)
        if len(streams) > 1:
            offs[1:] = np.cumsum(lens)[:-1]
        total = int(lens.sum())
        dev = self.volume.device
        stream = stream if stream is not None else torch.cuda.current_stream(dev)
        self._ensure(max(total, 1), stream)
        host = self._host.numpy()
        if total:
            np.concatenate(streams, out=host[:total])
        with torch.cuda.device(dev), torch.cuda.stream(stream):
            # copy, index uploads, event and staging kernel all on the caller's stream
            if total:
                self._dev[:total].copy_(self._host[:total], non_blocking=True)
                self._ev = torch.cuda.Event()
                self._ev.record()
            b_t = torch.as_tensor(np.asarray(bricks, dtype=np.int64)).to(dev, torch.int32)
            o_t = torch.as_tensor(offs).to(dev)
            l_t = torch.as_tensor(lens).to(dev, torch.int32)
            _lib.check(_lib.lib().csv_volume_stage_detail(
                self.volume._h, _ptr(b_t) if bricks else 0, _ptr(o_t) if bricks else 0, _ptr(l_t) if bricks else 0,
                len(bricks), _ptr(self._dev), total, _stream_handle(torch, stream)))
        self.staged_bytes_total += total
        self.staged_last_frame = total
