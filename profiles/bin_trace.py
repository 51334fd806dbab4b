"""K2 (bin_kernel) phase profile of CTA 0 from %globaltimer (FGS_FLAG_COUNTERS): microseconds spent
per phase, summed over the scatter's sub-ranges. Run on the GPU box: python profiles/bin_trace.py [cfg]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_04751_b200 import Rasterizer, RenderOptions, _lib, synthetic  # noqa: E402
from tests._helpers import to_device  # noqa: E402

NAMES = ["counts+rows+row hist", "compaction+offsets+row lists", "grid barriers", "scatter: zero counters",
         "scatter: count pass", "(fast: sub-chunk prefix)", "scatter: tile reservations", "scatter: key pass"]

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sc, deg, cams, _ = synthetic.config(cfg, **({"views": 1} if cfg >= 3 else {}))
r = Rasterizer(0)
ds = to_device(sc)
for _ in range(3):
    r.forward(ds, cams[0], RenderOptions(sh_degree=deg))
r.set_flags(_lib.FGS_FLAG_COUNTERS)
for _ in range(3):
    r.forward(ds, cams[0], RenderOptions(sh_degree=deg))
    torch.cuda.synchronize()
    t = r.debug("bin_trace", np.uint64).astype(np.int64)
    print(f"cfg{cfg} I={r.counts()['num_intersections']} " + "  ".join(f"{n}={v / 1000:.1f}us" for n, v in zip(NAMES, t)),
          f" total={t.sum() / 1000:.1f}us")
