"""Config-3 decode stage times without result checks (for A/B of deliberately wrong variants)."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2308_16619_b200 as p
vol = p.synth_voronoi((2048, 2048, 2048), 100, 2, True)
enc = p.compress_volume_device(vol, p.CompressionConfig(brick_log2=5))
del vol
torch.cuda.empty_cache()
gv = enc.to_volume()
out = torch.empty((2048, 2048, 2048), dtype=torch.int32, device="cuda")
res = torch.empty((gv.n_bricks, 4), dtype=torch.int64, device="cuda")
gv.decode(0, out=out, results=res)
gv.set_timing(True)
st = []
for _ in range(5):
    gv.decode(0, out=out, results=res)
    st.append(gv.last_timing())
print(os.environ.get("CSVGPU_LIB", "in-tree"), [round(min(s[i] for s in st), 3) for i in range(3)])
