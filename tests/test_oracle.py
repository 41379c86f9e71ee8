"""Pin the CPU oracle (oracle/) against vectors the REFERENCE produced (tests/golden/).

These run on CPU; they establish that the oracle the GPU tests compare
against is itself bit-exact with csvol on every fixture.
"""
import hashlib

import numpy as np
import pytest

from conftest import FUZZ, VOLUMES, fuzz_container_bytes, golden_bytes, golden_json, golden_volume, h16

COLS = {"palette_off": 0, "palette_len": 1, "coarse_off": 2, "coarse_bytes": 3, "coarse_nibbles": 4,
        "detail_off": 5, "detail_bytes": 6, "detail_nibbles": 7}


def test_known_answers(oracle):
    ka = golden_json("known_answers.json")
    for x, y, z, m in ka["morton_encode"]:
        assert oracle.morton_encode(x, y, z) == m
    assert oracle.rans_encode([], np.full(16, 256)).hex() == ka["rans_uniform_empty"] == "00008000"
    assert oracle.rans_encode(list(range(16)), np.full(16, 256)).hex() == ka["rans_uniform_range16"]
    for hist, counts in ka["quantize"]:
        assert oracle.quantize_counts(hist).tolist() == counts
    for case in ka["rans_cases"]:
        counts = np.array(case["counts"], np.uint16)
        assert oracle.quantize_counts(case["hist"]).tolist() == case["counts"]
        nib = np.frombuffer(bytes.fromhex(case["nibbles"]), np.uint8)
        enc = oracle.rans_encode(nib, counts)
        assert enc.hex() == case["encoded"]
        st, where, dec = oracle.rans_decode(enc, nib.size, counts)
        assert st == 0 and np.array_equal(dec, nib)
    # b=2 brick [A x7, B]
    pal, c, d = oracle.encode_brick(np.array([11] * 7 + [22], np.uint32), 1)
    assert pal.tolist() == ka["spec_b2"]["palette"]
    assert c.tolist() == ka["spec_b2"]["coarse"] and d.tolist() == ka["spec_b2"]["detail"]


@pytest.mark.parametrize("name", VOLUMES)
def test_encoder_bytes_identical(oracle, name):
    """oracle compress_volume == reference compress_volume, byte for byte."""
    vol = golden_volume(name)
    ref = golden_bytes(name)
    g = golden_json(f"decode_{name}.json")
    c = oracle.compress_volume(vol, brick_log2=g["brick_log2"], entropy=g["entropy"], threads=2)
    assert c.to_bytes() == ref


@pytest.mark.parametrize("name", VOLUMES)
def test_decode_matches_reference(oracle, name):
    g = golden_json(f"decode_{name}.json")
    c = oracle.Container.from_bytes(golden_bytes(name))
    N = g["brick_log2"]
    for t in range(N + 1):
        bad, res, vol = oracle.decompress_volume(c, t, threads=2)
        assert bad == -1
        assert h16(vol) == g["volume"][str(t)], (name, t)
    for i, per_t in g["bricks"].items():
        for t, exp in per_t.items():
            t = int(t)
            if t >= N:
                continue
            res, out = oracle.container_decode_brick(c, int(i), t)
            assert exp[0] == "ok" and res[0] == 0
            assert [h16(out), res[3], res[4]] == exp[1:], (name, i, t)
    if N <= 5:
        vol = golden_volume(name)
        _, _, dec = oracle.decompress_volume(c, 0, threads=2)
        assert np.array_equal(dec, vol.astype(np.uint32))


def _outcome(oracle, c, i, t):
    res, out = oracle.container_decode_brick(c, i, t)
    if res[0] == -1:
        return ["err", "empty palette"]
    if res[0] != 0:
        return ["err", oracle.error_message(res[0], res[1], res[2])]
    return ["ok", h16(out), res[3], res[4]]


@pytest.mark.parametrize("name", FUZZ)
def test_fuzz_errors_match_reference(oracle, name):
    base = golden_bytes(name)
    cases = golden_json(f"fuzz_{name}.json")
    assert len(cases) > 10
    for case in cases:
        c = oracle.Container.from_bytes(fuzz_container_bytes(base, case))
        if case["dir"]:
            c.directory[case["brick"], COLS[case["dir"][0]]] = case["dir"][1]
        for t, exp in case["outcomes"].items():
            assert _outcome(oracle, c, case["brick"], int(t)) == exp, (name, case, t)


def test_config1_container(oracle):
    cfg = golden_json("config1.json")
    with open(__import__("conftest").GOLDEN + "/config1.csv1", "rb") as f:
        data = f.read()
    assert hashlib.sha256(data).hexdigest()[:16] == cfg["container_sha"] == "cfb2549aabe04cca"
    c = oracle.Container.from_bytes(data)
    for t in range(6):
        bad, _, vol = oracle.decompress_volume(c, t)
        assert bad == -1 and h16(vol) == cfg["volume"][str(t)]


@pytest.mark.slow
def test_config1_generator_and_encoder(oracle):
    """gen_synthetic restatement reproduces the reference input; encoder reproduces its container."""
    cfg = golden_json("config1.json")
    vol = oracle.gen_synthetic(0, (256, 256, 256), 4000)
    assert hashlib.sha256(vol.astype("<u4").tobytes()).hexdigest()[:16] == cfg["input_sha"] == "70906f1c5d15fbda"
    c = oracle.compress_volume(vol, brick_log2=5)
    assert hashlib.sha256(c.to_bytes()).hexdigest()[:16] == cfg["container_sha"]
