"""CPU-only tests of the host side: format parsing, Morton/table helpers, cache
bookkeeping, and the C-ABI library's exported symbols (no device calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, VOLUMES, golden_bytes, golden_json


def test_library_exports_every_declared_symbol():
    import paper_2308_16619_b200._lib as L
    L.build()
    header = open(os.path.join(ROOT, "include", "csvgpu.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(csv_\w+)\s*\(", header, re.M))
    assert declared == set(L.EXPORTS)
    lib = ctypes.CDLL(L.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.csv_version() == 1


@pytest.mark.parametrize("name", VOLUMES)
def test_container_roundtrip_bytes(name):
    import paper_2308_16619_b200 as p
    data = golden_bytes(name)
    c = p.CsvContainer.from_bytes(data)
    assert c.to_bytes() == data
    assert len(c.head_bytes()) == 120 and data[:120] == c.head_bytes()


def test_container_errors():
    import paper_2308_16619_b200 as p
    data = golden_bytes("a_b3")
    with pytest.raises(p.CorruptStreamError, match="container header truncated"):
        p.CsvContainer.from_bytes(data[:50])
    with pytest.raises(p.CorruptStreamError, match="bad magic"):
        p.CsvContainer.from_bytes(b"XSV1" + data[4:])
    with pytest.raises(p.CorruptStreamError, match="container detail section truncated"):
        p.CsvContainer.from_bytes(data[:-1])


def test_morton_and_neighbors():
    import paper_2308_16619_b200 as p
    ka = golden_json("known_answers.json")
    for x, y, z, m in ka["morton_encode"]:
        assert p.morton_encode(x, y, z) == m
    for m, xyz in ka["morton_decode"]:
        assert list(p.morton_decode(m)) == xyz
    cfg = p.BrickConfig(3)
    for x, y, z, lvl, axis, exp in ka["outside_neighbor"]:
        nb = p.outside_neighbor(p.NodeCoord(x, y, z, lvl), axis, cfg)
        assert (None if nb is None else [nb.x, nb.y, nb.z]) == exp


def test_quantize_counts_matches_reference():
    import paper_2308_16619_b200 as p
    ka = golden_json("known_answers.json")
    for hist, counts in ka["quantize"]:
        assert p.quantize_counts(np.array(hist)).tolist() == counts
    for case in ka["rans_cases"]:
        assert p.quantize_counts(np.array(case["hist"])).tolist() == case["counts"]


def test_packed_decode_table():
    from paper_2308_16619_b200.rans import FrequencyTable, packed_decode_table
    counts = np.array([3061, 1021] + [1] * 14, np.uint16)
    tab = packed_decode_table(FrequencyTable(counts))
    sym = tab & 15
    assert np.array_equal(sym, np.repeat(np.arange(16), counts))
    assert np.all((tab >> 16) == counts[sym])


class _FakeDecode:
    def __init__(self, N):
        self.N = N
        self.calls = []

    def __call__(self, brick, lod):
        self.calls.append((brick, lod))
        return np.full(8 ** (self.N - lod), brick * 10 + lod, np.uint32)


def test_cache_plan_matches_serial_semantics():
    """plan_frame reproduces end_frame_assign's placements (cache.py:139-195)."""
    from paper_2308_16619_b200.cache import BrickCache
    rng = np.random.default_rng(0)
    N = 3
    for trial in range(30):
        a = BrickCache(64, N, pool_bytes=4096 * 4)
        b = BrickCache(64, N, pool_bytes=4096 * 4)
        for frame in range(6):
            reqs = [(int(rng.integers(0, 64)), int(rng.integers(0, N))) for _ in range(int(rng.integers(1, 20)))]
            a.begin_frame(); b.begin_frame()
            for br, lod in reqs:
                a.mark_used(br, lod); b.mark_used(br, lod)
            dec = _FakeDecode(N)
            try:
                pa = a.end_frame_assign(reqs, dec)
            except Exception as e:
                with pytest.raises(type(e)):
                    b.plan_frame(reqs)
                break
            pb, live = b.plan_frame(reqs)
            assert pa == pb
            assert np.array_equal(a.block_start, b.block_start) and np.array_equal(a.resident_lod, b.resident_lod)
            # live fills are exactly the placements still resident at frame end
            for br, lod, start in live:
                assert b.block_start[br] == start and b.resident_lod[br] == lod
            assert a.stats.decodes == b.stats.decodes


def test_device_buffer_check():
    """GpuVolume's guard on caller buffers (shape, element size, layout, device)."""
    import torch
    from paper_2308_16619_b200.device import _check_buffer
    cpu = torch.device("cpu")
    _check_buffer("out", torch.empty(2, 3, 4, dtype=torch.int32), cpu, 4, shape=(2, 3, 4))
    with pytest.raises(ValueError, match="shape"):
        _check_buffer("out", torch.empty(2, 3, 5, dtype=torch.int32), cpu, 4, shape=(2, 3, 4))
    with pytest.raises(ValueError, match="contiguous"):
        _check_buffer("out", torch.empty(2, 4, 3, dtype=torch.int32).transpose(1, 2), cpu, 4, shape=(2, 3, 4))
    with pytest.raises(ValueError, match="contiguous"):
        _check_buffer("out", torch.empty(2, 3, 4, dtype=torch.int64), cpu, 4, shape=(2, 3, 4))
    with pytest.raises(ValueError, match="at least"):
        _check_buffer("results", torch.empty(3, 4, dtype=torch.int64), cpu, 8, min_numel=16)
    with pytest.raises(ValueError, match="is on"):
        _check_buffer("out", torch.empty(1, dtype=torch.int32), torch.device("cuda", 0), 4)
