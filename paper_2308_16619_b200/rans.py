"""Static-table rANS format over the 16-symbol nibble alphabet (host side).

Format constants and table semantics follow csvol/rans.py:1-117: 32-bit
state, lower bound 2**23, byte renormalisation, 12-bit precision (counts sum
to 4096).  Table construction (histogram quantisation) stays on the host --
it is 16 numbers per volume.  Decoding runs on the GPU (K1 lanes in
csrc/csv_decode.cu); `packed_decode_table` is the layout those lanes read
from shared memory.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np

PRECISION_BITS = 12
TOTAL_FREQ = 1 << PRECISION_BITS
STATE_LOWER = 1 << 23
NUM_SYMBOLS = 16


@dataclass(frozen=True)
class FrequencyTable:
    """Quantised symbol counts (sum 4096) plus derived lookups (rans.py:31-62)."""

    counts: np.ndarray

    def __post_init__(self):
        counts = np.asarray(self.counts, dtype=np.uint16)
        if counts.shape != (NUM_SYMBOLS,):
            raise ValueError(f"expected {NUM_SYMBOLS} counts, got shape {counts.shape}")
        if int(counts.sum()) != TOTAL_FREQ:
            raise ValueError(f"counts must sum to {TOTAL_FREQ}, got {int(counts.sum())}")
        object.__setattr__(self, "counts", counts)

    @property
    def cumulative(self) -> np.ndarray:
        cum = np.zeros(NUM_SYMBOLS + 1, dtype=np.int64)
        np.cumsum(self.counts, out=cum[1:])
        return cum

    @property
    def slot_symbols(self) -> np.ndarray:
        return np.repeat(np.arange(NUM_SYMBOLS, dtype=np.uint8), self.counts)

    @classmethod
    def uniform(cls) -> "FrequencyTable":
        return cls(np.full(NUM_SYMBOLS, TOTAL_FREQ // NUM_SYMBOLS, dtype=np.uint16))


@dataclass(frozen=True)
class TablePair:
    interior: FrequencyTable
    leaf: FrequencyTable


def quantize_counts(histogram: np.ndarray) -> np.ndarray:
    """Counts summing to 4096, every symbol >= 1 (rans.py:73-91).

    The 4080 slots left after the floor of one are split in proportion to the
    histogram; leftover slots go to the largest fractional parts, lower
    symbol first on ties.
    """
    h = np.asarray(histogram, dtype=np.int64)
    if h.shape != (NUM_SYMBOLS,) or h.min() < 0:
        raise ValueError("histogram must be 16 non-negative counts")
    if h.sum() == 0:
        h = np.ones(NUM_SYMBOLS, dtype=np.int64)
    free = TOTAL_FREQ - NUM_SYMBOLS
    exact = (h * free) / float(h.sum())
    whole = np.floor(exact).astype(np.int64)
    frac = exact - whole
    short = free - int(whole.sum())
    rank = sorted(range(NUM_SYMBOLS), key=lambda s: (-frac[s], s))
    for s in rank[:short]:
        whole[s] += 1
    return (whole + 1).astype(np.uint16)


def build_frequency_tables(sample_streams: Iterable[tuple[np.ndarray, np.ndarray]]) -> TablePair:
    """Table pair from sampled (coarse, detail) raw nibble streams, +1 smoothed (rans.py:94-117)."""
    hi = np.zeros(NUM_SYMBOLS, dtype=np.int64)
    hl = np.zeros(NUM_SYMBOLS, dtype=np.int64)
    any_sample = False
    for coarse, detail in sample_streams:
        any_sample = True
        hi += np.bincount(np.asarray(coarse, dtype=np.int64), minlength=NUM_SYMBOLS)[:NUM_SYMBOLS]
        hl += np.bincount(np.asarray(detail, dtype=np.int64), minlength=NUM_SYMBOLS)[:NUM_SYMBOLS]
    if not any_sample:
        from .errors import ConfigError
        raise ConfigError("frequency table prepass needs at least one sampled brick")
    return TablePair(FrequencyTable(quantize_counts(hi + 1)), FrequencyTable(quantize_counts(hl + 1)))


def packed_decode_table(table: FrequencyTable) -> np.ndarray:
    """4096 x u32 {freq:16 | slot-cum:12 | symbol:4}, the K1 shared-memory layout."""
    out = np.empty(TOTAL_FREQ, dtype=np.uint32)
    cum = table.cumulative
    for s in range(NUM_SYMBOLS):
        f = int(table.counts[s])
        slots = np.arange(f, dtype=np.uint32)
        out[cum[s]: cum[s] + f] = (np.uint32(f) << np.uint32(16)) | (slots << np.uint32(4)) | np.uint32(s)
    return out


# ------------------------------------------------------------------ raw-nibble coder (GPU)
def _streams_on_device(torch, arrays):
    """Concatenate byte arrays into one device buffer: (buffer, offsets u64, sizes u32)."""
    sizes = np.array([a.size for a in arrays], dtype=np.uint32)
    offs = np.zeros(len(arrays), dtype=np.uint64)
    if len(arrays) > 1:
        offs[1:] = np.cumsum(sizes[:-1], dtype=np.uint64)
    flat = np.concatenate([np.asarray(a, dtype=np.uint8) for a in arrays] + [np.zeros(16, np.uint8)])
    dev = torch.device("cuda", torch.cuda.current_device())
    return (torch.from_numpy(flat).to(dev), torch.from_numpy(offs.view(np.int64)).to(dev),
            torch.from_numpy(sizes.view(np.int32)).to(dev), dev)


def rans_decode(data: bytes, n_symbols: int, table: FrequencyTable) -> np.ndarray:
    """Decode exactly ``n_symbols`` nibbles and verify stream integrity (rans.py:183-198).

    Runs on the GPU (csv_rans_decode, one lane per stream); the reference's
    CorruptStreamError messages for truncated and desynchronized streams.
    """
    from . import _lib
    from .errors import CorruptStreamError
    torch = _lib.require_cuda()
    n_symbols = int(n_symbols)
    if n_symbols < 0:
        raise ValueError("negative symbol count")
    raw = np.frombuffer(bytes(data), dtype=np.uint8)
    buf, off, nb, dev = _streams_on_device(torch, [raw])
    nsym = torch.tensor([n_symbols], dtype=torch.int32, device=dev)
    out = torch.empty(max(n_symbols, 1), dtype=torch.uint8, device=dev)
    out_off = torch.zeros(1, dtype=torch.int64, device=dev)
    status = torch.empty(2, dtype=torch.int32, device=dev)
    counts = np.ascontiguousarray(table.counts, dtype=np.uint16)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().csv_rans_decode(buf.data_ptr(), off.data_ptr(), nb.data_ptr(), nsym.data_ptr(), 1,
                                              counts.ctypes.data, out.data_ptr(), out_off.data_ptr(),
                                              status.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    st, pos = (int(v) for v in status.cpu().tolist())
    if st == 1:
        raise CorruptStreamError(f"entropy stream truncated at symbol {pos}")
    if st == 2:
        raise CorruptStreamError(f"entropy stream desynchronized after {n_symbols} symbols")
    return out[:n_symbols].cpu().numpy()


def rans_encode(nibbles, table: FrequencyTable) -> bytes:
    """Entropy-code a nibble sequence; deterministic and byte-exact (rans.py:168-180).

    The encodability check is the reference's (host); the coding runs on the
    GPU (csv_rans_encode)."""
    from . import _lib
    from .errors import EncodabilityError
    torch = _lib.require_cuda()
    arr = np.ascontiguousarray(nibbles, dtype=np.uint8)
    counts = np.ascontiguousarray(table.counts, dtype=np.uint16)
    if arr.size and (arr.max() >= NUM_SYMBOLS or counts[np.minimum(arr, 15)].min() == 0):
        bad = int(np.flatnonzero((arr >= NUM_SYMBOLS) | (counts[np.minimum(arr, 15)] == 0))[0])
        raise EncodabilityError(f"nibble {int(arr[bad])} at position {bad} has zero frequency")
    buf, off, _, dev = _streams_on_device(torch, [arr])
    nsym = torch.tensor([arr.size], dtype=torch.int32, device=dev)
    cap = 2 * arr.size + 8
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    out_off = torch.zeros(1, dtype=torch.int64, device=dev)
    start = torch.empty(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().csv_rans_encode(buf.data_ptr(), off.data_ptr(), nsym.data_ptr(), 1, counts.ctypes.data,
                                              out.data_ptr(), out_off.data_ptr(), start.data_ptr(),
                                              torch.cuda.current_stream(dev).cuda_stream))
    s0 = int(start.item())
    return out[s0:cap].cpu().numpy().tobytes()

