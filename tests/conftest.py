"""Shared fixtures.  `-m gpu` tests need a CUDA device; everything else runs on CPU."""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

VOLUMES = ["a_b3", "b_b1", "c_b2_mem", "d_b5_mem", "e_b4_raw", "f_b2_noise", "g_b6", "h_b3_u16", "i_const",
           "j_b7", "k_b5_noise_raw", "l_b4_bigval"]
FUZZ = ["a_b3", "c_b2_mem", "d_b5_mem", "e_b4_raw", "f_b2_noise", "g_b6"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def h16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4").tobytes()).hexdigest()[:16]


def golden_bytes(name: str) -> bytes:
    with open(os.path.join(GOLDEN, f"vol_{name}.csv1"), "rb") as f:
        return f.read()


def golden_volume(name: str) -> np.ndarray:
    return np.load(os.path.join(GOLDEN, f"vol_{name}.npz"))["volume"]


def golden_json(fname: str):
    with open(os.path.join(GOLDEN, fname)) as f:
        return json.load(f)


def fuzz_container_bytes(base: bytes, case) -> bytes:
    data = bytearray(base)
    for off, x in case["xor"]:
        data[off] ^= x
    return bytes(data)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc
    orc.build()
    return orc
