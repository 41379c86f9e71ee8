"""GPU encoder parity: containers byte-identical to the reference's compress_volume."""
import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, VOLUMES, golden_bytes, golden_json, golden_volume, h16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_16619_b200 as p
    return p


@pytest.mark.parametrize("name", VOLUMES)
def test_encoder_bytes_identical(pkg, name):
    g = golden_json(f"decode_{name}.json")
    vol = golden_volume(name)
    c = pkg.compress_volume(vol, pkg.CompressionConfig(brick_log2=g["brick_log2"], entropy=g["entropy"]))
    assert c.to_bytes() == golden_bytes(name)


def test_encoder_config1(pkg, oracle):
    cfg = golden_json("config1.json")
    vol = oracle.gen_synthetic(0, (256, 256, 256), 4000)
    c = pkg.compress_volume(vol, pkg.CompressionConfig(brick_log2=5))
    data = c.to_bytes()
    assert hashlib.sha256(data).hexdigest()[:16] == cfg["container_sha"] == "cfb2549aabe04cca"


@pytest.mark.parametrize("bl2,entropy,stride", [(5, True, 512), (4, True, 7), (3, False, 512), (6, True, 3)])
def test_device_roundtrip_voronoi(pkg, oracle, bl2, entropy, stride):
    """synth -> GPU encode -> GPU decode == input; host container == oracle encoder bytes."""
    import torch
    d = pkg.synth_voronoi((150, 130, 97), 6, seed=11, membrane=True)
    enc = pkg.compress_volume_device(d, pkg.CompressionConfig(brick_log2=bl2, entropy=entropy, prepass_stride=stride))
    vol = enc.to_volume()
    out = pkg.decompress_volume_device(vol, 0)
    assert torch.equal(out, d)
    host = d.cpu().numpy().view(np.uint32)
    ref = oracle.compress_volume(host, brick_log2=bl2, entropy=entropy, prepass_stride=stride)
    assert enc.to_container().to_bytes() == ref.to_bytes()
    for t in range(1, bl2 + 1):
        got = pkg.decompress_volume_device(vol, t).cpu().numpy().view(np.uint32)
        bad, _, exp = oracle.decompress_volume(ref, t)
        assert bad == -1 and np.array_equal(got, exp), t


def test_synth_deterministic(pkg):
    import torch
    a = pkg.synth_voronoi((64, 48, 40), 5, seed=3, membrane=True)
    b = pkg.synth_voronoi((64, 48, 40), 5, seed=3, membrane=True)
    assert torch.equal(a, b)
    assert int((a == 0).sum()) > 0 and int(a.max()) <= 125


@pytest.mark.parametrize("membrane,drift", [(True, 0.0), (False, 0.0), (True, 1.0)])
def test_synth_matches_oracle(pkg, oracle, membrane, drift):
    d = pkg.synth_voronoi((70, 50, 33), 6, seed=9, membrane=membrane, drift=drift, drift_seed=4)
    ref = oracle.synth_voronoi((70, 50, 33), 6, seed=9, membrane=membrane, drift=drift, drift_seed=4)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), ref)
    part = oracle.synth_voronoi((70, 50, 33), 6, seed=9, membrane=membrane, drift=drift, drift_seed=4, z_range=(10, 20))
    assert np.array_equal(part, ref[10:20])


def test_concurrent_encodes_share_the_scratch_arena(pkg):
    """Encodes from several host threads (ctypes drops the GIL) serialise on the
    per-device scratch arena and each still produces the reference's bytes; the
    arena grows from a small b=3 encode to b=5 and back."""
    from concurrent.futures import ThreadPoolExecutor
    names = ["a_b3", "d_b5_mem", "g_b6", "j_b7"] * 2
    cases = []
    for n in names:
        g = golden_json(f"decode_{n}.json")
        cases.append((n, golden_volume(n), pkg.CompressionConfig(brick_log2=g["brick_log2"], entropy=g["entropy"])))

    def run(case):
        n, vol, cfg = case
        return n, pkg.compress_volume(vol, cfg).to_bytes()

    with ThreadPoolExecutor(max_workers=4) as ex:
        for n, data in ex.map(run, cases):
            assert data == golden_bytes(n), n
