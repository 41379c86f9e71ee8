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


def test_oracle_dropin_goldens(oracle):
    """The oracle's rANS coder, pyramid and per-brick encoder against the reference's
    own outputs for the stand-alone drop-ins (tests/golden/dropin.json)."""
    import os
    from conftest import GOLDEN, golden_json, h16
    G = golden_json("dropin.json")
    for case in G["rans"]:
        counts = np.array(case["counts"], dtype=np.uint16)
        nib = np.frombuffer(bytes.fromhex(case["nibbles"]), dtype=np.uint8)
        data = bytes.fromhex(case["encoded"])
        assert oracle.rans_encode(nib, counts) == data
        st, where, out = oracle.rans_decode(data, nib.size, counts)
        assert st == 0 and h16(out) == case["decode"]["exact"]["ok"]
        st, where, _ = oracle.rans_decode(data[:-1], nib.size, counts)
        exp = case["decode"]["short"]
        if "error" in exp:
            assert st == 1 and exp["error"] == f"entropy stream truncated at symbol {where}"
    for case, enc in zip(G["pyramid"], G["encode"]):
        N = case["brick_log2"]
        src = case["source"]
        if "labels" in src:
            flat = np.frombuffer(bytes.fromhex(src["labels"]), dtype="<u4").astype(np.uint32)
        else:
            vol = np.load(os.path.join(GOLDEN, f"vol_{src['vol']}.npz"))["volume"]
            b = 1 << N
            z, y, x = src["zyx"]
            grid = np.zeros((b, b, b), dtype=np.uint32)
            piece = vol[z:z + b, y:y + b, x:x + b]
            grid[:piece.shape[0], :piece.shape[1], :piece.shape[2]] = piece
            flat = np.empty(b ** 3, dtype=np.uint32)
            flat[oracle.morton_codes(b)] = grid.ravel()
        assert [h16(oracle.pyramid_level(flat, N, t)) for t in range(N + 1)] == case["levels"], case["name"]
        pal, co, de = oracle.encode_brick(flat, N)
        assert (h16(pal), pal.size, h16(co), co.size, h16(de), de.size) == \
            (enc["palette"], enc["n_palette"], enc["coarse"], enc["n_coarse"], enc["detail"], enc["n_detail"])
