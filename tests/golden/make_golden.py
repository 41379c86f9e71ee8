"""Generate the golden parity fixtures from the REFERENCE implementation.

Run once in the survey/build container (the reference is importable only
there; it does not travel to the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs (all under tests/golden/):
  known_answers.json        Morton / rANS / quantizer known answers
  vol_<name>.npz            small input volumes (compressed)
  vol_<name>.csv1           the reference's container for that volume
  decode_<name>.json        per-(brick, t) decode results of the reference:
                            sha256[:16] of the Morton output and consumed counts,
                            plus the decompress_volume hash per t
  fuzz_<name>.json          corrupted-stream cases: mutation + the reference's
                            outcome (message, or output hash and consumed counts)
  config1.json              config-1 input/container/decoded hashes
  config1.csv1              the reference's config-1 container (1.28 MB)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import csvol
from csvol import codec, container as cvol, morton, rans
from csvol.errors import CorruptStreamError

OUT = os.path.dirname(os.path.abspath(__file__))


def h16(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4").tobytes()).hexdigest()[:16]


def membranes(vol: np.ndarray) -> np.ndarray:
    """Label 0 on voxels whose +x/+y/+z neighbour differs (thin boundaries)."""
    v = vol.copy()
    edge = np.zeros(v.shape, bool)
    edge[:, :, :-1] |= vol[:, :, :-1] != vol[:, :, 1:]
    edge[:, :-1, :] |= vol[:, :-1, :] != vol[:, 1:, :]
    edge[:-1, :, :] |= vol[:-1, :, :] != vol[1:, :, :]
    v[edge] = 0
    return v


def volumes():
    rng = np.random.default_rng(1234)
    vols = {}
    vols["a_b3"] = (csvol.gen_synthetic(1, (40, 36, 28), 60), 3, True)
    vols["b_b1"] = (csvol.gen_synthetic(2, (9, 7, 5), 6), 1, True)
    vols["c_b2_mem"] = (membranes(csvol.gen_synthetic(3, (30, 20, 17), 25)), 2, True)
    vols["d_b5_mem"] = (membranes(csvol.gen_synthetic(4, (70, 64, 40), 90)), 5, True)
    vols["e_b4_raw"] = (membranes(csvol.gen_synthetic(5, (33, 33, 17), 40)), 4, False)
    vols["f_b2_noise"] = (rng.integers(0, 300, (13, 11, 9)).astype(np.uint32), 2, True)
    vols["g_b6"] = (membranes(csvol.gen_synthetic(6, (70, 64, 64), 30)), 6, True)
    vols["h_b3_u16"] = (csvol.gen_synthetic(7, (17, 16, 15), 20).astype(np.uint16), 3, True)
    vols["i_const"] = (np.full((20, 20, 20), 77, np.uint32), 3, True)
    vols["j_b7"] = (membranes(csvol.gen_synthetic(8, (130, 24, 12), 12)), 7, True)
    vols["k_b5_noise_raw"] = ((rng.integers(0, 40, (32, 32, 32)) * 1000003).astype(np.uint32), 5, False)
    vols["l_b4_bigval"] = ((csvol.gen_synthetic(9, (16, 16, 16), 30).astype(np.uint64) * 143000011 % 2**32).astype(np.uint32), 4, True)
    return vols


def brick_results(cont, i, t):
    """Reference decode of brick i at LOD t: ('ok', hash, ci, di) or ('err', message)."""
    N = cont.meta.brick_log2
    try:
        out = cont.decode_brick(i, t)
    except CorruptStreamError as e:
        return ["err", str(e)]
    ci = di = 0
    if t < N:
        entry = cont.directory[i]
        if cont.meta.entropy:
            det = cont.brick_detail(i) if t == 0 else np.empty(0, np.uint8)
            nd = int(entry["detail_nibbles"]) if t == 0 else 0
            _, ci, di = codec.decode_brick_entropy(cont.brick_palette(i), cont.brick_coarse(i),
                                                   int(entry["coarse_nibbles"]), det, nd, cont.tables, t,
                                                   cont.config, return_consumed=True)
        else:
            enc = codec.BrickEncoding(N, cont.brick_palette(i),
                                      cvol._unpack_nibbles(cont.brick_coarse(i), int(entry["coarse_nibbles"])),
                                      cvol._unpack_nibbles(cont.brick_detail(i) if t == 0 else np.empty(0, np.uint8),
                                                           int(entry["detail_nibbles"]) if t == 0 else 0))
            _, ci, di = codec.decode_brick(enc, t, cont.config, return_consumed=True)
    return ["ok", h16(out), int(ci), int(di)]


def known_answers():
    ka = {}
    ka["morton_encode"] = [[x, y, z, csvol.morton_encode(x, y, z)] for x, y, z in
                           [(3, 5, 1), (0, 0, 1), (1, 0, 0), (31, 31, 31), (7, 0, 3), (100, 200, 300)]]
    ka["morton_decode"] = [[m, list(csvol.morton_decode(m))] for m in [7, 143, 4, 12345, 2**20 + 5]]
    ka["outside_neighbor"] = []
    cfg = morton.BrickConfig(3)
    for (x, y, z, lvl, axis) in [(0, 0, 0, 0, "x"), (2, 3, 5, 0, "x"), (5, 2, 0, 0, "y"), (7, 7, 7, 0, "z"),
                                 (1, 1, 1, 1, "z"), (3, 0, 2, 1, "x")]:
        nb = morton.outside_neighbor(morton.NodeCoord(x, y, z, lvl), axis, cfg)
        ka["outside_neighbor"].append([x, y, z, lvl, axis, None if nb is None else [nb.x, nb.y, nb.z]])
    uni = rans.FrequencyTable.uniform()
    ka["rans_uniform_empty"] = rans.rans_encode([], uni).hex()
    ka["rans_uniform_range16"] = rans.rans_encode(list(range(16)), uni).hex()
    rng = np.random.default_rng(99)
    cases = []
    for k in range(40):
        hist = rng.integers(0, 1000, 16) * (rng.random(16) < 0.7)
        counts = rans.quantize_counts(hist)
        n = int(rng.integers(0, 400))
        p = counts / counts.sum()
        nib = rng.choice(16, size=n, p=p).astype(np.uint8)
        enc = rans.rans_encode(nib, rans.FrequencyTable(counts))
        cases.append({"hist": hist.tolist(), "counts": counts.tolist(), "nibbles": nib.tobytes().hex(),
                      "encoded": enc.hex()})
    ka["rans_cases"] = cases
    ka["quantize"] = [[[3, 1] + [0] * 14, rans.quantize_counts(np.array([3, 1] + [0] * 14)).tolist()],
                      [[0] * 16, rans.quantize_counts(np.zeros(16, np.int64)).tolist()],
                      [[1] * 16, rans.quantize_counts(np.ones(16, np.int64)).tolist()],
                      [[5, 5, 5] + [0] * 13, rans.quantize_counts(np.array([5, 5, 5] + [0] * 13)).tolist()]]
    # SPEC.md:174 example: b=2 brick [A x7, B]
    A, B = 11, 22
    grid = np.array([A] * 7 + [B], np.uint32)
    enc = codec.encode_brick(csvol.build_pyramid(grid, morton.BrickConfig(1)))
    ka["spec_b2"] = {"palette": enc.palette.tolist(), "coarse": enc.coarse.tolist(), "detail": enc.detail.tolist()}
    return ka


def mutate_cases(name, cont, blob, n_cases, rng, t_values):
    """Corrupt one brick per case; record the reference outcome for each t."""
    base = cont.to_bytes()
    head = cvol._HEADER.size + 64 + cvol._BLOBS.size
    n = cont.meta.brick_count
    dir_off = head
    pal_off = head + n * cvol.DIRECTORY_DTYPE.itemsize
    c_off = pal_off + cont.palette_blob.size * 4
    d_off = c_off + cont.coarse_blob.size
    cases = []
    kinds = ["flip_coarse", "flip_detail", "flip_palette_len", "nib_coarse", "nib_detail", "bytes_coarse",
             "bytes_detail", "flip_coarse2", "flip_detail2"]
    tries = 0
    while len(cases) < n_cases and tries < 50 * n_cases:
        tries += 1
        i = int(rng.integers(0, n))
        e = cont.directory[i]
        kind = kinds[int(rng.integers(0, len(kinds)))]
        muts = []   # (absolute byte offset, xor mask)
        dirfix = None  # (field, new value)
        if kind.startswith("flip_coarse"):
            nb = int(e["coarse_bytes"])
            if nb == 0:
                continue
            for _ in range(1 if kind == "flip_coarse" else 3):
                muts.append([c_off + int(e["coarse_off"]) + int(rng.integers(0, nb)), 1 << int(rng.integers(0, 8))])
        elif kind.startswith("flip_detail"):
            nb = int(e["detail_bytes"])
            if nb == 0:
                continue
            for _ in range(1 if kind == "flip_detail" else 3):
                muts.append([d_off + int(e["detail_off"]) + int(rng.integers(0, nb)), 1 << int(rng.integers(0, 8))])
        elif kind == "flip_palette_len":
            dirfix = ["palette_len", max(0, int(e["palette_len"]) - int(rng.integers(1, 4)))]
        elif kind == "nib_coarse":
            dirfix = ["coarse_nibbles", max(0, int(e["coarse_nibbles"]) + int(rng.integers(-5, 6)))]
        elif kind == "nib_detail":
            dirfix = ["detail_nibbles", max(0, int(e["detail_nibbles"]) + int(rng.integers(-5, 6)))]
        elif kind == "bytes_coarse":
            dirfix = ["coarse_bytes", max(0, int(e["coarse_bytes"]) - int(rng.integers(1, 6)))]
        elif kind == "bytes_detail":
            dirfix = ["detail_bytes", max(0, int(e["detail_bytes"]) - int(rng.integers(1, 6)))]
        data = bytearray(base)
        for off, x in muts:
            data[off] ^= x
        c2 = csvol.CsvContainer.from_bytes(bytes(data))
        if dirfix is not None:
            d = c2.directory.copy()
            d[i][dirfix[0]] = dirfix[1]
            c2.directory = d
        outcomes = {str(t): brick_results(c2, i, t) for t in t_values}
        cases.append({"brick": i, "kind": kind, "xor": muts, "dir": dirfix, "outcomes": outcomes})
    return cases


def main():
    ka = known_answers()
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(ka, f, indent=1)
    rng = np.random.default_rng(4321)
    for name, (vol, bl2, entropy) in volumes().items():
        cont = csvol.compress_volume(vol, csvol.CompressionConfig(brick_log2=bl2, entropy=entropy, workers=1))
        data = cont.to_bytes()
        with open(os.path.join(OUT, f"vol_{name}.csv1"), "wb") as f:
            f.write(data)
        np.savez_compressed(os.path.join(OUT, f"vol_{name}.npz"), volume=vol)
        N = bl2
        res = {"brick_log2": N, "entropy": entropy, "shape": list(vol.shape), "dtype": str(vol.dtype),
               "container_sha": hashlib.sha256(data).hexdigest()[:16], "bricks": {}, "volume": {}}
        for t in range(N + 1):
            res["volume"][str(t)] = h16(csvol.decompress_volume(cont, t))
        nb = cont.meta.brick_count
        for i in range(nb):
            res["bricks"][str(i)] = {str(t): brick_results(cont, i, t) for t in range(N + 1)}
        with open(os.path.join(OUT, f"decode_{name}.json"), "w") as f:
            json.dump(res, f)
        if name in ("a_b3", "c_b2_mem", "d_b5_mem", "e_b4_raw", "g_b6", "f_b2_noise"):
            ncase = {"d_b5_mem": 240, "g_b6": 40}.get(name, 80)
            tv = list(range(min(N, 3)))
            cases = mutate_cases(name, cont, data, ncase, rng, tv)
            with open(os.path.join(OUT, f"fuzz_{name}.json"), "w") as f:
                json.dump(cases, f)
        print(name, len(data), nb, flush=True)
    # config 1
    vol = csvol.gen_synthetic(0, (256, 256, 256), 4000)
    cont = csvol.compress_volume(vol, csvol.CompressionConfig(brick_log2=5, workers=8))
    data = cont.to_bytes()
    with open(os.path.join(OUT, "config1.csv1"), "wb") as f:
        f.write(data)
    cfg = {"input_sha": hashlib.sha256(vol.astype("<u4").tobytes()).hexdigest()[:16],
           "container_sha": hashlib.sha256(data).hexdigest()[:16], "container_bytes": len(data),
           "volume": {str(t): h16(csvol.decompress_volume(cont, t, workers=8)) for t in range(6)},
           "bricks_sampled": {}}
    for i in range(0, cont.meta.brick_count, 37):
        cfg["bricks_sampled"][str(i)] = {str(t): brick_results(cont, i, t) for t in range(6)}
    with open(os.path.join(OUT, "config1.json"), "w") as f:
        json.dump(cfg, f, indent=1)
    print("config1", cfg["input_sha"], cfg["container_sha"], len(data))


if __name__ == "__main__" and not os.environ.get("CSV_GOLDEN_STATS"):
    sys.exit(main())


def make_stats_goldens():
    """stats() of the reference for a few golden containers."""
    out = {}
    for name in ("a_b3", "d_b5_mem", "e_b4_raw", "f_b2_noise", "i_const", "g_b6"):
        with open(os.path.join(OUT, f"vol_{name}.csv1"), "rb") as f:
            c = csvol.CsvContainer.from_bytes(f.read())
        out[name] = cvol.stats(c)
    with open(os.path.join(OUT, "config1.csv1"), "rb") as f:
        out["config1"] = cvol.stats(csvol.CsvContainer.from_bytes(f.read()))
    with open(os.path.join(OUT, "stats.json"), "w") as f:
        json.dump(out, f, indent=1, default=lambda o: list(o) if isinstance(o, tuple) else o)


if __name__ == "__main__" and os.environ.get("CSV_GOLDEN_STATS"):
    make_stats_goldens()
