"""K3 / forward stage times (ms per frame, CUDA events on every frame) at config 2 for the library
FGS_LIB selects (A/B of the per-tile sort paths).   python profiles/k3probe.py"""
# K3 alone: time blend_forward via the library's stage events over many frames (cfg2), for the lib in FGS_LIB
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2409_04751_b200 import Rasterizer, RenderOptions, synthetic, _lib
from tests._helpers import to_device
sc, deg, cams, _ = synthetic.config(2)
ds = to_device(sc); r = Rasterizer(0); o = RenderOptions(sh_degree=deg)
for _ in range(10): r.forward(ds, cams[0], o)
torch.cuda.synchronize()
r.set_flags(_lib.FGS_FLAG_TIMING); r.timing(reset=True)
for _ in range(200): r.forward(ds, cams[0], o)
torch.cuda.synchronize()
t = r.timing(reset=True)
n = t["forward_calls"]
print(os.environ.get("FGS_LIB", "base"), os.environ.get("FGS_FWD_PX", "-"), {k: round(v / n, 4) for k, v in t["ms"].items() if v})
