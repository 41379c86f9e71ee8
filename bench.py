#!/usr/bin/env python
"""Benchmark of the B200 CSV decode path: decoded GVoxel/s, HBM roofline, e2e, CPU baseline.

Workload (BASELINE.json north_star / configs[2]):
  synthetic 2048^3 jittered-grid Voronoi, ~1M labels (100^3 cells), 1-voxel
  label-0 membranes, seed 2; brick 32^3, rANS on, prepass stride 512.
  The volume is generated and encoded on the GPU (byte-identical to the
  reference encoder, tests/test_gpu_encode.py) before timing.

One step = one full-volume decode at LOD 0 of this rank's brick range (K1
entropy lanes + K2 replay/raster writer) from HBM-resident compressed data
into an HBM-resident (Z,Y,X) uint32 output.  Output (34 GB) and input
(~0.9 GB) both exceed the 126 MB L2, so no flush is needed between steps.

Multi-GPU (--gpus N under torchrun), north_star's configuration by default
(--scaling strong): ONE 2048^3 volume, its brick index range-partitioned in
whole bz layers over the ranks (distributed.rank_bricks); value = 2048^3 /
max-over-ranks decode time.  The decoded slabs' gather to rank 0 (grouped
ncclSend/ncclRecv into the root's volume) and to every rank
(all_gather_into_tensor) are timed separately ("decode_gather").
--scaling weak (one volume per rank) is kept as a labelled extra.

`--impl reference` times the reference itself (csvol from baseline/_ref, its
numba decoder through decompress_volume(workers=all host cores)) on a bounded
sample of the same workload; the oracle's C port is timed beside it.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "config3": dict(dims=(2048, 2048, 2048), cells=100, seed=2, membrane=True,
                    desc="config 3: 2048^3 Voronoi, 100^3 cells (~1M labels), 1-voxel label-0 membranes, seed 2"),
    "config2": dict(dims=(1024, 1024, 1024), cells=22, seed=1, membrane=False,
                    desc="config 2: 1024^3 cell-like Voronoi, 22^3 cells (~10k labels), seed 1"),
}
BRICK_LOG2 = 5


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cache", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/e2e/cpu)")
    ap.add_argument("--zlayers", type=int, default=0, help="profiling: only the first K bz-layers of the volume")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): one volume range-partitioned over the ranks; weak: one volume per rank")
    ap.add_argument("--no-gather", action="store_true", help="skip the decode+gather timing")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower().startswith("active")})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------- distributed
def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours":
        torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: int, world: int) -> int:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.int64, device="cuda")
    dist.all_reduce(t)
    return int(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------- CPU baselines
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def import_csvol():
    """The reference package from baseline/_ref (pip --target install of /root/reference),
    or (None, why)."""
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "csvol_numba_cache"))
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "csvol")):
        return None, "baseline/_ref/csvol not installed"
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import csvol
        import csvol.cli
        return csvol, None
    except Exception as e:   # numba missing etc.
        return None, f"{type(e).__name__}: {e}"


def sample_volume(wl, layers: int, cores: int):
    """First `layers` bz-layers of the workload's volume (oracle generator, same field as the GPU one)."""
    from oracle import oracle as orc
    orc.build()
    X, Y, Z = wl["dims"]
    zs = min(layers << BRICK_LOG2, Z)
    # rows [0, zs] (+1 row so membranes of the last row see their +z neighbour)
    return orc.synth_voronoi((X, Y, Z), wl["cells"], wl["seed"], wl["membrane"],
                             z_range=(0, min(zs + 1, Z)), threads=cores)[:zs]


def port_decode_baseline(wl, cores: int, layers: int = 8, reps: int = 3):
    """The oracle's C restatement of _decode_kernel + morton_to_grid, OpenMP over bricks."""
    from oracle import oracle as orc
    vol = sample_volume(wl, layers, cores)
    c = orc.compress_volume(np.ascontiguousarray(vol), brick_log2=BRICK_LOG2, threads=cores)
    X, Y, _ = wl["dims"]
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        bad, _, _ = orc.decompress_volume(c, 0, threads=cores)
        times.append(time.perf_counter() - t0)
        assert bad == -1
    vox = vol.size
    return {"value": vox / min(times) / 1e9, "unit": "GVoxel/s", "cores": cores, "kind": "port",
            "sample": f"first {layers} bz-layer(s) ({X}x{Y}x{vol.shape[0]} = {vox / 1e6:.0f} MVox); "
                      f"oracle/ C port of _decode_kernel + morton_to_grid, {cores} OpenMP threads, best of {reps}"}, c


def csvol_container(csvol, orc_container):
    return csvol.CsvContainer.from_bytes(orc_container.to_bytes())


def reference_decode(csvol, c, vox: int, workers: int, reps: int):
    """csvol.decompress_volume(c, 0, workers=W) timed as cli.py:125-169 times it
    (JIT warmed by cli._warm_kernels, perf_counter, best of reps)."""
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        csvol.decompress_volume(c, 0, workers=workers)
        times.append(time.perf_counter() - t0)
    return vox / min(times) / 1e9, times


def reference_cache_frame(csvol, c, reqs, n_sample: int):
    """Config 4 on the reference's own path: BrickCache.end_frame_assign with
    CsvContainer.decode_brick as the decode hook (cache.py:139-170,
    render.py:876-885), serial by construction, on the first n_sample requests."""
    sub = reqs[:n_sample]
    cache = csvol.BrickCache(c.meta.brick_count, BRICK_LOG2, pool_bytes=4 << 30)
    cache.begin_frame()
    for b, l in sub:
        cache.mark_used(b, l)
    t0 = time.perf_counter()
    placed = cache.end_frame_assign(sub, lambda b, l: c.decode_brick(b, l))
    dt = time.perf_counter() - t0
    vox = sum(8 ** (BRICK_LOG2 - l) for _, l in placed)
    return {"value": vox / dt / 1e9, "unit": "GVoxel/s", "requests": len(sub), "seconds": dt,
            "us_per_brick": dt / max(len(sub), 1) * 1e6,
            "sample": f"the {len(sub)} nearest of config 4's 65,536 requests (all in the first bz-layers), "
                      f"one end_frame_assign into an empty pool, serial"}


def reference_compress(csvol, wl5, cores: int, layers: int = 1):
    """Config 5 encode on the reference: compress_volume(workers=all) (container.py:374-453)
    on the first bz-layer(s) of timestep 0."""
    from oracle import oracle as orc
    X, Y, Z = wl5["dims"]
    zs = min(layers << BRICK_LOG2, Z)
    vol = orc.synth_voronoi((X, Y, Z), wl5["cells"], wl5["seed"], False, z_range=(0, zs), threads=cores)
    t0 = time.perf_counter()
    csvol.compress_volume(vol, csvol.CompressionConfig(brick_log2=BRICK_LOG2, workers=cores))
    dt = time.perf_counter() - t0
    return {"value": vol.size / dt / 1e9, "unit": "GVoxel/s", "seconds": dt, "cores": cores,
            "sample": f"compress_volume of the first {layers} bz-layer(s) of a config-5 timestep "
                      f"({X}x{Y}x{zs}), workers={cores}"}


def cpu_baselines(wl, cache_reqs=None):
    """Every CPU number the line carries (rank 0, N=1): the reference (csvol) decoder at
    W = all cores (the headline baseline) and W = 1, its cache path (config 4) and
    encoder (config 5), and the oracle's C port."""
    cores = len(os.sched_getaffinity(0))
    out = {"cpu_model": cpu_model()}
    port, pc = port_decode_baseline(wl, cores)
    csvol, why = import_csvol()
    if csvol is None:
        port["reference_unavailable"] = why
        port["cpu_model"] = out["cpu_model"]
        return port
    csvol.cli._warm_kernels()
    X, Y, _ = wl["dims"]
    from oracle import oracle as orc
    vol2 = sample_volume(wl, 2, cores)
    c2 = csvol_container(csvol, orc.compress_volume(np.ascontiguousarray(vol2), brick_log2=BRICK_LOG2, threads=cores))
    vall, tall = reference_decode(csvol, c2, vol2.size, cores, 3)
    vol1 = vol2[: 1 << BRICK_LOG2]
    c1 = csvol_container(csvol, orc.compress_volume(np.ascontiguousarray(vol1), brick_log2=BRICK_LOG2, threads=cores))
    v1, t1 = reference_decode(csvol, c1, vol1.size, 1, 1)
    line = {"value": vall, "unit": "GVoxel/s", "cores": cores, "kind": "reference",
            "sample": f"first 2 bz-layers ({X}x{Y}x{vol2.shape[0]} = {vol2.size / 1e6:.0f} MVox); "
                      f"csvol.decompress_volume(c, 0, workers={cores}) from baseline/_ref (numba, JIT warmed), "
                      f"best of 3: {[round(x, 3) for x in tall]} s",
            "cpu_model": out["cpu_model"],
            "w1": {"value": v1, "unit": "GVoxel/s", "cores": 1, "seconds": t1[0],
                   "sample": f"first bz-layer ({vol1.size / 1e6:.0f} MVox), workers=1"},
            "port": port}
    if cache_reqs:
        line["cache_path"] = reference_cache_frame(csvol, c2, [r for r in cache_reqs if r[0] < c2.meta.brick_count],
                                                   4096)
    line["compress"] = reference_compress(csvol, WORKLOADS["config2"] | {"seed": 3}, cores)
    return line


def run_reference(args, world, rank):
    """The reference arm: csvol's own decoder (baseline/_ref) on the host cores, W + K
    steps of one decompress_volume(workers=all) over a 2-bz-layer sample each."""
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    cores = len(os.sched_getaffinity(0))
    X, Y, Z = wl["dims"]
    csvol, why = import_csvol()
    from oracle import oracle as orc
    vol = sample_volume(wl, 2, cores)
    oc = orc.compress_volume(np.ascontiguousarray(vol), brick_log2=BRICK_LOG2, threads=cores)
    if csvol is not None:
        csvol.cli._warm_kernels()
        c = csvol_container(csvol, oc)
        step = lambda: csvol.decompress_volume(c, 0, workers=cores)   # noqa: E731
        kind, what = "reference", f"csvol.decompress_volume(c, 0, workers={cores}) (baseline/_ref, numba)"
    else:
        step = lambda: orc.decompress_volume(oc, 0, threads=cores)   # noqa: E731
        kind, what = "port", f"oracle C port, {cores} OpenMP threads (csvol unavailable: {why})"
    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    ms = statistics.mean(times) * 1e3
    value = vol.size / (ms * 1e-3) / 1e9
    sample = (f"each step decodes the first 2 bz-layers of the workload ({X}x{Y}x{vol.shape[0]} = "
              f"{vol.size / 1e6:.0f} MVox of the {X * Y * Z / 1e6:.0f} MVox volume); {what}")
    line = {"impl": "reference", "metric": "decoded GVoxel/s (full-volume decode, LOD 0)", "value": value,
            "unit": "GVoxel/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": wl["desc"], "brick": 32, "entropy": "rANS", "lod": 0,
                       "bricks": int(np.prod([-(-d // 32) for d in wl["dims"]])),
                       "sample_voxels_per_step": int(vol.size)},
            "step_seconds": [round(x, 4) for x in times],
            "cpu_baseline": {"value": value, "unit": "GVoxel/s", "cores": cores, "kind": kind, "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "GVoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- config 4 requests
def desired_lods(grid, b, cam, fov, height, max_lod):
    """render.py:145-158 restated: per-brick LOD from brick-centre distance."""
    gx, gy, gz = grid
    idx = np.arange(gx * gy * gz)
    cx = (idx % gx + 0.5) * b
    cy = (idx // gx % gy + 0.5) * b
    cz = (idx // (gx * gy) + 0.5) * b
    d = np.sqrt((cx - cam[0]) ** 2 + (cy - cam[1]) ** 2 + (cz - cam[2]) ** 2)
    ratio = np.maximum(1.0, d * 2.0 * math.tan(fov / 2.0) / height)
    lod = np.clip(np.ceil(np.log2(ratio)).astype(np.int64), 0, max_lod)
    return lod, d


# ---------------------------------------------------------------------------- config 5
def timeseries_leg(p, torch, dev, stream, world: int = 1, rank: int = 0, total: int = 16,
                   dims=(1024, 1024, 1024), cells: int = 22):
    """16 timesteps of 1024^3 Voronoi (seed 3, seeds drifting
    by <= k voxels at step k) sharded over the ranks (rank r takes timesteps r, r + N, ...;
    2 per rank at N = 8, 16 on one GPU); per timestep GPU encode then GPU decode, both
    timed with CUDA events (the decode after one untimed call that allocates the new
    volume's workspace; one untimed encode + decode before the first timestep); lossless
    round trip checked (untimed).  Ensemble throughput =
    16 * 1024^3 voxels / the slowest rank's summed encode (decode) time."""
    enc_ms, dec_ms = [], []
    X, Y, Z = dims
    mine = list(range(rank, total, world))
    # warm-up (untimed): one encode + decode, so that kernel loading and the encoder's
    # one-time scratch arena / memory-pool growth are not charged to the first timestep
    vol = p.synth_voronoi(dims, cells, seed=3, membrane=False, drift=0.0, drift_seed=3, device=dev)
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=BRICK_LOG2))
    gv = enc.to_volume()
    out = torch.empty_like(vol)
    gv.decode(0, out=out)
    torch.cuda.synchronize()
    gv.close()
    enc.close()
    del vol, out
    for k in mine:
        vol = p.synth_voronoi(dims, cells, seed=3, membrane=False, drift=float(min(k, 16)), drift_seed=3 + k,
                              device=dev)
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=BRICK_LOG2))
        e1.record(stream)
        gv = enc.to_volume()
        out = torch.empty_like(vol)
        gv.decode(0, out=out)               # untimed: sizes this volume's decode workspace (one-off cudaMalloc)
        torch.cuda.synchronize()
        e1b = torch.cuda.Event(enable_timing=True)
        e1b.record(stream)
        gv.decode(0, out=out)
        e2.record(stream)
        torch.cuda.synchronize()
        assert torch.equal(out, vol), "time-series round trip mismatch"
        enc_ms.append(e0.elapsed_time(e1))
        dec_ms.append(e1b.elapsed_time(e2))
        gv.close()
        enc.close()
        del vol, out
        torch.cuda.empty_cache()
    te = max_over_ranks(sum(enc_ms) / 1e3, world)
    td = max_over_ranks(sum(dec_ms) / 1e3, world)
    vox = X * Y * Z * total
    return {"timesteps": total, "per_rank": len(mine), "dims": list(dims), "encode_gvox_s": vox / te / 1e9,
            "decode_gvox_s": vox / td / 1e9, "roundtrip_gvox_s": vox / (te + td) / 1e9,
            "encode_ms_rank0": [round(x, 2) for x in enc_ms], "decode_ms_rank0": [round(x, 3) for x in dec_ms],
            "workload": f"config 5: {total} timesteps of 1024^3 Voronoi (22^3 cells, seed 3, drift <= k) over "
                        f"{world} GPU(s), rank r takes timesteps r, r + N, ...; max over ranks of the summed "
                        "CUDA-event times"}


# ---------------------------------------------------------------------------- our arm
def strong_rank_plan(dims, brick_log2: int, world: int, rank: int) -> dict:
    """This rank's share of ONE volume (north_star / SURVEY.md §8e): whole bz layers,
    contiguous brick range and LOD-0 raster rows."""
    from paper_2308_16619_b200.distributed import rank_bricks, rank_slab
    X, Y, Z = dims
    b = 1 << brick_log2
    grid = (-(-X // b), -(-Y // b), -(-Z // b))
    b0, b1 = rank_bricks(grid, world, rank)
    z0, z1 = rank_slab(dims, brick_log2, 0, world, rank)
    return {"bricks": (b0, b1), "rows": (z0, z1), "layers": (b0 // (grid[0] * grid[1]), b1 // (grid[0] * grid[1])),
            "voxels": (z1 - z0) * Y * X}


def sample_bricks(vol, grid, n: int = 64, seed: int = 7):
    """A fixed sample of brick indices with their raster blocks (cropped), kept on the host
    to verify the timed output after the run."""
    gx, gy, gz = grid
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, gx * gy * gz - 1], rng.integers(0, gx * gy * gz, n - 2)]))
    b = 1 << BRICK_LOG2
    blocks = {}
    for i in idx.tolist():
        bx, by, bz = i % gx, i // gx % gy, i // (gx * gy)
        blocks[i] = vol[bz * b:(bz + 1) * b, by * b:(by + 1) * b, bx * b:(bx + 1) * b].cpu()
    return blocks


def check_bricks(blocks, out, z_first: int, brick_lo: int, brick_hi: int, grid) -> dict:
    """Compare the sampled bricks inside [brick_lo, brick_hi) with `out` (rows from z_first)."""
    gx, gy, _ = grid
    b = 1 << BRICK_LOG2
    n = bad = 0
    for i, ref in blocks.items():
        if not brick_lo <= i < brick_hi:
            continue
        bx, by, bz = i % gx, i // gx % gy, i // (gx * gy)
        got = out[bz * b - z_first:(bz + 1) * b - z_first, by * b:(by + 1) * b, bx * b:(bx + 1) * b].cpu()
        n += 1
        bad += 0 if torch_equal(got, ref) else 1
    return {"bricks_checked": n, "mismatches": bad}


def torch_equal(a, b) -> bool:
    import torch
    return a.shape == b.shape and bool(torch.equal(a, b))


def run_ours(args, world, rank, local):
    import torch
    import paper_2308_16619_b200 as p
    from paper_2308_16619_b200.distributed import gather_slabs
    wl = dict(WORKLOADS[args.workload])
    if args.zlayers:
        wl["dims"] = (wl["dims"][0], wl["dims"][1], 32 * args.zlayers)
        wl["desc"] += f" (first {args.zlayers} bz-layers only)"
    X, Y, Z = wl["dims"]
    dev = torch.device("cuda", local)
    hbm, peak_kind = peaks()
    b = 1 << BRICK_LOG2
    grid = gx, gy, gz = (-(-X // b), -(-Y // b), -(-Z // b))
    weak = args.scaling == "weak"
    # ---- data: GPU synth + GPU encode (untimed); strong: every rank builds the same volume
    t0 = time.perf_counter()
    seed = wl["seed"] + (rank if weak else 0)
    vol = p.synth_voronoi((X, Y, Z), wl["cells"], seed, wl["membrane"], device=dev)
    torch.cuda.synchronize()
    t_synth = time.perf_counter() - t0
    blocks = sample_bricks(vol, grid)
    t0 = time.perf_counter()
    enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=BRICK_LOG2))
    torch.cuda.synchronize()
    t_enc = time.perf_counter() - t0
    del vol
    torch.cuda.empty_cache()
    plan = strong_rank_plan((X, Y, Z), BRICK_LOG2, 1 if weak else world, 0 if weak else rank)
    brick_range = plan["bricks"]
    zr = plan["rows"]
    gv = enc.to_volume(brick_range)
    root = rank == 0
    # the root holds the whole volume (strong) and decodes its slab straight into its rows
    full = None
    if not weak and root:
        full = torch.empty((Z, Y, X), dtype=torch.int32, device=dev)
        out = full[zr[0]:zr[1]]
    else:
        out = torch.empty((zr[1] - zr[0], Y, X), dtype=torch.int32, device=dev)
    res = torch.empty((max(gv.n_bricks, 1), 4), dtype=torch.int64, device=dev)
    voxels_rank = plan["voxels"]
    voxels_all = X * Y * Z * (world if weak else 1)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        gv.decode(0, out=out, results=res)
    torch.cuda.synchronize()
    p.GpuVolume.raise_first(res, gv.n_bricks)
    # ---- timed region: decode only
    clocks = Clocks(local)
    if not args.profile:
        clocks.start()
        time.sleep(0.3)
    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        gv.decode(0, out=out, results=res)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    clk = clocks.stop() if not args.profile else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["profile"]}
    p.GpuVolume.raise_first(res, gv.n_bricks)
    ms = max_over_ranks(ms_rank, world)
    value = voxels_all / (ms * 1e-3) / 1e9
    check = check_bricks(blocks, out, zr[0], brick_range[0], brick_range[1], grid)
    # ---- decode + gather (strong): the slabs to the root's volume (grouped send/recv), and
    # to every rank (all_gather_into_tensor); at N = 1 the gather is a no-op
    gather = None
    if not weak and not args.no_gather and not args.profile:
        gather = {}
        for mode in ("root", "all"):
            if mode == "all" and world > 1 and not root:
                vol_all = torch.empty((Z, Y, X), dtype=torch.int32, device=dev)
            else:
                vol_all = full
            dst = vol_all[zr[0]:zr[1]] if vol_all is not None and (mode == "all" or root) else out

            def step():
                gv.decode(0, out=dst, results=res)
                if world > 1:
                    gather_slabs(dst, vol_all if (mode == "all" or root) else None, (X, Y, Z), BRICK_LOG2, 0,
                                 mode=mode, root=0)
            step()
            torch.cuda.synchronize()
            barrier(world)
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(args.steps):
                step()
            g1.record(stream)
            torch.cuda.synchronize()
            barrier(world)
            gms = max_over_ranks(g0.elapsed_time(g1) / args.steps, world)
            ent = {"value": X * Y * Z / (gms * 1e-3) / 1e9, "unit": "GVoxel/s", "ms_per_step": gms,
                   "gather_bytes_per_rank": 4 * (X * Y * Z - voxels_rank) if mode == "all" else
                   (4 * (X * Y * Z - voxels_rank) if root else 4 * voxels_rank),
                   "collective": ("none (N = 1)" if world == 1 else
                                  "batch_isend_irecv: grouped ncclSend/ncclRecv of each slab into the root's "
                                  "(Z,Y,X) rows" if mode == "root" else
                                  "all_gather_into_tensor into each rank's (Z,Y,X) volume")}
            if mode == "root" and root:
                ent["check"] = check_bricks(blocks, full, 0, 0, gx * gy * gz, grid)
            gather[mode] = ent
            if mode == "all" and world > 1 and not root:
                del vol_all
                torch.cuda.empty_cache()
        # fused decode + gather through peer memory (distributed.PeerVolume): the root's volume
        # is mapped by every rank (CUDA IPC; NVLink P2P across GPUs) and each rank's K2w stores
        # its rows straight into it -- the transfer overlaps the decode, no NCCL data movement
        from paper_2308_16619_b200.distributed import PeerVolume
        if root:
            pv = PeerVolume.alloc((Z, Y, X), dev)
        if world > 1:
            import torch.distributed as tdist
            box = [pv.handle if root else None]
            tdist.broadcast_object_list(box, src=0)
            if not root:
                pv = PeerVolume.open(box[0], (Z, Y, X), dev)
        pptr = pv.rows_ptr(zr[0])
        gv.decode_into(0, pptr, zr, res)
        torch.cuda.synchronize()
        barrier(world)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            gv.decode_into(0, pptr, zr, res)
        g1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        gms = max_over_ranks(g0.elapsed_time(g1) / args.steps, world)
        ent = {"value": X * Y * Z / (gms * 1e-3) / 1e9, "unit": "GVoxel/s", "ms_per_step": gms,
               "gather_bytes_per_rank": 0 if root else 4 * voxels_rank,
               "collective": ("none (N = 1): decode into an IPC-shareable volume" if world == 1 else
                              "none: every rank's K2w stores its rows into the root's volume through CUDA IPC "
                              "peer memory (NVLink P2P); max-over-ranks decode time with the stores landed")}
        if root:
            ent["check"] = check_bricks(blocks, pv.tensor(), 0, 0, gx * gy * gz, grid)
        gather["peer"] = ent
        pv.close()
        del pv
    # ---- per-stage timing (CUDA events on the launching stream, separate pass)
    gv.set_timing(True)
    stages = []
    for _ in range(3):
        gv.decode(0, out=out, results=res)
        stages.append(gv.last_timing())
    gv.set_timing(False)
    plan_ms, k1_ms, k2_ms = (statistics.median(s[i] for s in stages) for i in range(3))
    # ---- algorithmic bytes for this rank's bricks, split by kernel:
    # K1 reads the coarse/detail streams + directory, K2w the palettes + directory and
    # writes the voxels.  K1's entry bytes are an intermediate and count for neither.
    cont = enc.to_container()
    d = cont.directory[brick_range[0]:brick_range[1]]
    pal_b = 4 * int(d["palette_len"].sum())
    cb_b = int(d["coarse_bytes"].sum())
    db_b = int(d["detail_bytes"].sum())
    n_b = brick_range[1] - brick_range[0]
    step_bytes = pal_b + cb_b + db_b + 44 * n_b + 64 + 4 * voxels_rank
    k1_bytes = cb_b + db_b + 44 * n_b + 64
    k2_bytes = pal_b + 44 * n_b + 4 * voxels_rank
    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("workload") == args.workload and not args.zlayers and (world == 1 or weak):
            traffic = tj
    except Exception:
        pass

    def kline(name, kms, kbytes):
        ach = kbytes / (kms * 1e-3) / 1e9
        return {"bound": "hbm", "kernel": name, "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic.get(name), "peak_kind": peak_kind, "algorithmic_bytes": kbytes, "kernel_ms": kms}
    kernels = {"k1_streams": kline("k1_streams", k1_ms, k1_bytes), "k2_warp": kline("k2_warp", k2_ms, k2_bytes)}
    roofline = dict(kernels["k2_warp"] if k2_ms >= k1_ms else kernels["k1_streams"])
    long_pal = int(d["palette_len"].max()) > 253 if n_b else False      # K2w runs a second (u16) pass (e8::kMarkPal)
    step_gbs = step_bytes / (ms_rank * 1e-3) / 1e9
    line = {
        "metric": "decoded GVoxel/s (full-volume decode, LOD 0)", "value": value, "unit": "GVoxel/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (GPU Voronoi generator; GPU encoder, byte-identical to the reference encoder)",
        "config": {"workload": wl["desc"], "brick": 32, "entropy": "rANS", "lod": 0, "bricks": gx * gy * gz,
                   "compressed_bytes": int(enc.payload_bytes), "compression_rate": enc.payload_bytes / (4 * X * Y * Z),
                   "parallelism": (f"one config-3 volume per rank (seed {wl['seed']} + rank) x{world}" if weak
                                   else f"one volume, bz layers [{plan['layers'][0]}, {plan['layers'][1]}) on rank "
                                        f"{rank} of {world} (whole-bz-layer brick ranges)"),
                   "l2": "inputs (~%.1f GB compressed) and output (%.1f GB) exceed L2; no flush" %
                         (enc.payload_bytes / 1e9, 4 * X * Y * Z / 1e9)},
        "roofline": roofline,
        "kernels": kernels,
        "step_roofline": {"achieved": step_gbs, "peak": hbm, "unit": "GB/s", "frac": step_gbs / hbm,
                          "algorithmic_bytes": step_bytes, "bytes_per_voxel": step_bytes / voxels_rank},
        "stages_ms": {"plan": plan_ms, "k1_streams": k1_ms, "k2_replay": k2_ms},
        "clocks": clk,
        "gpu_launches": (7 if long_pal else 6) * args.steps,   # sizes, 3 scan, K1, K2w (+ u16 K2w)
        "check": dict(check, what="sampled bricks of the timed output vs the generated input volume"),
        "setup_s": {"synth": t_synth, "encode": t_enc},
    }
    if gather is not None:
        line["decode_gather"] = gather
    # ---- e2e: public API, host buffers in, host volume out (pinned)
    if not args.no_e2e and not args.profile:
        try:                                   # one pinned 34 GB volume per rank; pageable if the host refuses
            pin = torch.empty((zr[1] - zr[0], Y, X), dtype=torch.int32, pin_memory=True)
        except RuntimeError:
            pin = torch.empty((zr[1] - zr[0], Y, X), dtype=torch.int32)
        times = []
        pin_np = pin.numpy().view(np.uint32)
        layers = None if weak else plan["layers"]
        # the step's inputs in pinned host memory (the container's blobs copied once, untimed):
        # the H2D copies inside the timed region are then DMA, not CPU-staged pageable copies
        # that block the enqueueing thread and compete with the D2H for host DRAM bandwidth
        def pinned_copy(a):
            t_ = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
            v_ = t_.numpy().view(a.dtype)
            v_[...] = a.reshape(-1)
            return t_, v_
        pins_in = [pinned_copy(a) for a in (cont.palette_blob, cont.coarse_blob, cont.detail_blob)]
        cont_h = dataclasses.replace(cont, palette_blob=pins_in[0][1], coarse_blob=pins_in[1][1],
                                     detail_blob=pins_in[2][1])
        # one untimed call first: the freshly pinned pages' first device writes (IOMMU / page
        # setup) cost the first one or two calls up to 2x
        p.decompress_volume(cont_h, 0, out=pin_np, layers=layers)
        for it in range(5):
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            # the reference-facing API, host container in / host (slab of the) volume out
            p.decompress_volume(cont_h, 0, out=pin_np, layers=layers)
            times.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(min(times), world)
        h2d = sum_over_ranks(44 * n_b + pal_b + cb_b + db_b, world)
        d2h = sum_over_ranks(4 * voxels_rank, world)
        line["e2e"] = {"value": voxels_all / e2e_s / 1e9, "unit": "GVoxel/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "seconds": e2e_s,
                       "seconds_all": [round(x, 4) for x in times],
                       "reduction": "best of 5 after one untimed call (host-timed, synchronised), max over ranks",
                       "path": "decompress_volume(container with pinned blobs, 0, out=pinned host array%s): H2D of directory+blobs, "
                               "slab-pipelined GPU decode overlapped with D2H into the pinned (Z,Y,X) uint32 %s" %
                               (", layers=this rank's bz range" if layers else "",
                                "slab of each rank" if layers and world > 1 else "volume")}
        e2e_check = check_bricks(blocks, pin, zr[0], brick_range[0], brick_range[1], grid)
        line["e2e"]["check"] = e2e_check
        del pin, pins_in, cont_h
        torch.cuda.synchronize()
        torch.cuda.empty_cache()   # the slab buffers (2 x 4.3 GB) back to the device before the cache legs
    # ---- config 4: batched random-access decode into a device brick pool
    cache_reqs = None
    if not args.no_cache and not args.profile and (world == 1 or not weak):
        lod, dist = desired_lods((gx, gy, gz), b, (1024.0, 1024.0, -64.0), math.pi / 3, 1080, BRICK_LOG2)
        order = np.argsort(dist, kind="stable")[:65536]
        reqs = [(int(i), int(lod[i])) for i in order if lod[i] < BRICK_LOG2]
        cache_reqs = reqs
        if world > 1:   # strong: each rank serves the requests of the bricks it owns (no collective)
            reqs = [r for r in reqs if brick_range[0] <= r[0] < brick_range[1]]
        cache = p.BrickCache(gx * gy * gz, BRICK_LOG2, pool_bytes=8 << 30, device=dev)
        cache.begin_frame()
        for br, l in reqs:
            cache.mark_used(br, l)
        tp0 = time.perf_counter()
        placed, live = cache.plan_frame(reqs)
        host_plan_ms = (time.perf_counter() - tp0) * 1e3
        arr = np.asarray(live, dtype=np.int64)
        bricks = torch.from_numpy(arr[:, 0].astype(np.int32)).to(dev)
        lods = torch.from_numpy(arr[:, 1].astype(np.uint8)).to(dev)
        dst = torch.from_numpy(arr[:, 2] * 8).to(dev)
        fvol = enc.to_volume() if world == 1 else gv
        cres = torch.empty((max(len(live), 1), 4), dtype=torch.int64, device=dev)
        for _ in range(args.warmup):
            fvol.decode_bricks(bricks, lods, dst, cache.pool, results=cres)
        torch.cuda.synchronize()
        p.GpuVolume.raise_first(cres, len(live))
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fvol.decode_bricks(bricks, lods, dst, cache.pool, results=cres)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        cms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        cvox = sum_over_ranks(int(sum(8 ** (BRICK_LOG2 - int(l)) for l in arr[:, 1])) if len(arr) else 0, world)
        n0 = sum_over_ranks(int((arr[:, 1] == 0).sum()) if len(arr) else 0, world)
        nreq = sum_over_ranks(len(live), world)
        line["random_brick"] = {"value": cvox / (cms * 1e-3) / 1e9, "unit": "GVoxel/s", "ms_per_step": cms,
                                "requests": nreq, "lod0": n0, "lod1": nreq - n0, "voxels": cvox,
                                "workload": "config 4: camera (1024,1024,-64) +z, H=1080, fov pi/3, "
                                            "desired_lods, 65,536 nearest bricks -> BrickCache plan -> one "
                                            "csv_decode_bricks batch into an 8 GiB device pool"
                                            + (f"; requests partitioned by brick owner over {world} ranks, "
                                               "max-over-ranks time" if world > 1 else "")}
        if world > 1:
            del cache
            torch.cuda.empty_cache()
    if cache_reqs is not None and world == 1:
        # the same frame with the residency bookkeeping on the GPU too:
        # device LOD selection + DeviceBrickCache (evict / free stacks / carve, atomics) + batched decode
        del cache
        torch.cuda.empty_cache()
        dcache = p.DeviceBrickCache(gx * gy * gz, BRICK_LOG2, pool_bytes=8 << 30, device=dev)
        rb = torch.from_numpy(np.array([r[0] for r in reqs], np.int32)).to(dev)
        rl = torch.from_numpy(np.array([r[1] for r in reqs], np.uint8)).to(dev)
        none_b = torch.empty(0, dtype=torch.int32, device=dev)
        none_l = torch.empty(0, dtype=torch.uint8, device=dev)
        cam = p.Camera(position=(1024.0, 1024.0, -64.0), fov=math.pi / 3, width=1920, height=1080)
        dl = p.desired_lods_device(fvol, cam)
        assert torch.equal(dl[rb.long()], rl), "device LODs differ from the restated desired_lods"

        def frame():
            p.desired_lods_device(fvol, cam, out=dl)
            dcache.begin_frame()
            dcache.mark_used(rb, rl)
            return dcache.end_frame_assign(rb, rl, fvol)

        def evict_all():
            dcache.begin_frame()
            dcache.end_frame_assign(none_b, none_l, fvol)

        for _ in range(max(1, args.warmup)):
            evict_all()
            frame()
        ftimes = []
        for _ in range(args.steps):
            evict_all()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nplaced = frame()
            torch.cuda.synchronize()
            ftimes.append(time.perf_counter() - t0)
        fs = statistics.median(ftimes)
        line["random_brick"]["device_frame"] = {
            "value": cvox / fs / 1e9, "unit": "GVoxel/s", "ms_per_frame": fs * 1e3, "placed": nplaced,
            "host_plan_ms": host_plan_ms,   # the reference-style serial bookkeeping of the same frame (cache.py)
            "path": "desired_lods_device + DeviceBrickCache begin_frame/mark_used/end_frame_assign "
                    "(want, free stacks, carve, batched K1+K2w decode); wall clock, median"}
        # cold detail: the detail blob stays in host memory, 8 MiB of
        # requested level-0 streams staged per frame, the rest decoded at level 1
        hostc = enc.to_container()
        cold = hostc.to_device(device=dev, cold_detail=True)
        dstream = p.DeviceDetailStream(hostc, cold, budget_bytes=8 << 20)
        reqs_np = np.asarray(reqs, dtype=np.int64)
        ctimes, cvox_c, nstaged = [], 0, 0
        for it in range(max(1, args.warmup) + args.steps):
            evict_all()
            dstream.hot.clear()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            adj_b, adj_l = dstream.plan_arrays(reqs_np)
            ab = torch.from_numpy(adj_b.astype(np.int32)).to(dev)
            al = torch.from_numpy(adj_l.astype(np.uint8)).to(dev)
            dcache.begin_frame()
            dcache.mark_used(ab, al)
            dcache.end_frame_assign(ab, al, cold, detail=dstream)
            torch.cuda.synchronize()
            if it >= max(1, args.warmup):
                ctimes.append(time.perf_counter() - t0)
            cvox_c = int((8 ** (BRICK_LOG2 - adj_l)).sum())
            nstaged = dstream.staged_last_frame
        cs = statistics.median(ctimes)
        line["random_brick"]["cold_detail_frame"] = {
            "value": cvox_c / cs / 1e9, "unit": "GVoxel/s", "ms_per_frame": cs * 1e3,
            "budget_bytes": 8 << 20, "staged_bytes": nstaged, "deferred_to_lod1": dstream.deferred_last_frame,
            "path": "DetailStore.plan_arrays (8 MiB budget) + DeviceBrickCache plan + one pinned H2D of the fetched "
                    "level-0 streams + batched decode; detail blob never resident on the GPU; wall clock, median"}
        cold.close()
        dcache.close()
        fvol.close()
    # ---- config 5: the 16-timestep ensemble encode + decode, timesteps sharded over the ranks
    if not args.no_cache and not args.profile and args.workload == "config3" and not args.zlayers:
        line["timeseries"] = timeseries_leg(p, torch, dev, stream, world, rank)
    if not args.no_cpu and not args.profile and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baselines(wl, cache_reqs)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
