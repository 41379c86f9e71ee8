"""Fused decode + gather through peer memory (distributed.decompress_volume_peer):
two ranks as two processes on ONE device (gloo for the control messages, a
CUDA IPC buffer for the data -- the same calls map NVLink peer memory when the
ranks own different GPUs).  Rank 1 decodes its bz layers straight into rank 0's
volume; rank 0 checks the whole volume against the reference's hashes; a
corrupted container raises the same message on both ranks."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

WORKER = r"""
import os, sys, json, hashlib
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, %(root)r); sys.path.insert(0, %(here)r)
import paper_2308_16619_b200 as p
from paper_2308_16619_b200.distributed import decompress_volume_peer
from conftest import golden_bytes, golden_json, h16
rank = int(sys.argv[1])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%(port)d", rank=rank, world_size=2)
torch.cuda.set_device(0)
out = {}
for name in ("d_b5_mem", "a_b3"):
    g = golden_json("decode_%%s.json" %% name)
    c = p.CsvContainer.from_bytes(golden_bytes(name))
    for t in range(g["brick_log2"] + 1):
        pv = decompress_volume_peer(c, t)
        if rank == 0:
            out["%%s/%%d" %% (name, t)] = h16(pv.tensor().cpu().numpy().view(np.uint32)) == g["volume"][str(t)]
            pv.close()
        else:
            assert pv is None
# corrupted: truncate the detail stream of the last brick (owned by rank 1)
c = p.CsvContainer.from_bytes(golden_bytes("d_b5_mem"))
d = c.directory.copy(); d[-1]["detail_bytes"] = 2; c.directory = d
try:
    decompress_volume_peer(c, 0)
    out["err"] = None
except p.CorruptStreamError as e:
    out["err"] = str(e)
print("RESULT", rank, json.dumps(out))
dist.destroy_process_group()
"""


def test_peer_gather_two_ranks_one_device(tmp_path):
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    code = WORKER % {"root": os.path.dirname(HERE), "here": HERE, "port": port}
    script = tmp_path / "peer_worker.py"
    script.write_text(code)
    procs = [subprocess.Popen([sys.executable, str(script), str(r)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(2)]
    outs = [pr.communicate(timeout=600) for pr in procs]
    res = {}
    for pr, (o, e) in zip(procs, outs):
        assert pr.returncode == 0, e[-3000:]
        line = [l for l in o.splitlines() if l.startswith("RESULT")][-1]
        _, r, js = line.split(" ", 2)
        import json
        res[int(r)] = json.loads(js)
    checks = {k: v for k, v in res[0].items() if k != "err"}
    assert checks and all(checks.values()), checks
    assert res[0]["err"] is not None and res[0]["err"] == res[1]["err"]
