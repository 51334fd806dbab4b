"""Quick probe: forward stage times + blend counters (E_eval, E_contrib, culled evals, max CTA
cycles) for a config on cuda:0."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg=2, reps=20):
    import torch

    from paper_2409_04751_b200 import BackwardOptions, Rasterizer, RenderOptions, _lib, synthetic
    from tests._helpers import to_device

    sc, deg, cams, dls = synthetic.config(cfg)
    ds = to_device(sc)
    r = Rasterizer(0)
    o = RenderOptions(sh_degree=deg)
    r.set_flags(_lib.FGS_FLAG_COUNTERS)
    for _ in range(3):
        r.forward(ds, cams[0], o)
    torch.cuda.synchronize()
    c = r.debug("counters", np.uint64)
    print(f"COUNTERS e_eval={c[0]} e_contrib={c[1]} culled_evals={int(c[2])} max_cta_us={c[3] / 1965.0:.1f}")
    r.set_flags(_lib.FGS_FLAG_TIMING)
    dl = torch.from_numpy(dls[0]).cuda() if dls else torch.randn((cams[0].height, cams[0].width, 3), device="cuda")
    for _ in range(2):  # warm-up: first launches of each kernel variant pay lazy module loading
        r.forward(ds, cams[0], o)
        r.backward(ds, cams[0], dl, BackwardOptions())
    torch.cuda.synchronize()
    r.timing(reset=True)
    for _ in range(reps):
        r.forward(ds, cams[0], o)
        r.backward(ds, cams[0], dl, BackwardOptions())
    t = r.timing()
    print("STAGES_US", {k: round(1000 * v / reps, 1) for k, v in t["ms"].items()})




def bin_trace(cfg=2):
    import torch

    from paper_2409_04751_b200 import Rasterizer, RenderOptions, _lib, synthetic
    from tests._helpers import to_device

    sc, deg, cams, _ = synthetic.config(cfg)
    ds = to_device(sc)
    r = Rasterizer(0)
    r.set_flags(_lib.FGS_FLAG_COUNTERS)
    for _ in range(3):
        r.forward(ds, cams[0], RenderOptions(sh_degree=deg))
    torch.cuda.synchronize()
    t = r.debug("bin_trace", np.uint64).astype(np.int64)
    names = ["compact", "pass0", "pass1", "pass2", "pass3", "rankscan"]
    l1 = [(names[i], (t[i + 1] - t[i]) / 1000.0) for i in range(6)]
    l2n = ["duplicate", "tilesort", "ranges+gather", "sync", "order"]
    l2 = [(l2n[i], (t[9 + i] - t[8 + i]) / 1000.0) for i in range(5)]
    print("BIN_TRACE_US level1", l1, "level2", l2)
    p = t[16:22]
    print("PASS1_US", [("hist", (p[0] - t[2]) / 1e3), ("sync1", (p[1] - p[0]) / 1e3), ("colscan", (p[2] - p[1]) / 1e3),
                       ("sync2", (p[3] - p[2]) / 1e3), ("rank+scatter", (p[4] - p[3]) / 1e3), ("sync3", (p[5] - p[4]) / 1e3)])


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
    bin_trace(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
