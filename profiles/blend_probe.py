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
    r.timing(reset=True)
    dl = torch.from_numpy(dls[0]).cuda() if dls else torch.randn((cams[0].height, cams[0].width, 3), device="cuda")
    for _ in range(reps):
        r.forward(ds, cams[0], o)
        r.backward(ds, cams[0], dl, BackwardOptions())
    t = r.timing()
    print("STAGES_US", {k: round(1000 * v / reps, 1) for k, v in t["ms"].items()})


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
