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
