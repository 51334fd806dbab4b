import numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_2409_04751_b200 import Rasterizer, RenderOptions, synthetic, _lib
from tests._helpers import to_device
for cfg in (2,3):
    sc, deg, cams, _ = synthetic.config(cfg)
    r = Rasterizer(0); ds = to_device(sc)
    for _ in range(3): r.forward(ds, cams[0], RenderOptions(sh_degree=deg))
    r.set_flags(_lib.FGS_FLAG_COUNTERS)
    r.forward(ds, cams[0], RenderOptions(sh_degree=deg)); torch.cuda.synchronize()
    c = r.debug("counters16", np.uint64).astype(np.float64)
    tc = r.debug("tile_cycles", np.uint64).astype(np.float64)
    ntiles = c[7]; nbig = c[6]
    print(cfg, "tiles", ntiles, "big", nbig, "avg small sort cycles", c[4]/max(1,ntiles-nbig), "avg big sort cycles", c[5]/max(1,nbig),
          "total sort cycles", c[4]+c[5], "total CTA cycles", tc.sum(), "frac", (c[4]+c[5])/tc.sum())
