"""Driver for compute-sanitizer runs (tests/test_sanitizer.py and by hand): forward + backward of
one BASELINE config on cuda:0 through the C ABI, twice (the second frame takes the speculative
launch path), then a host-buffer render. Exits 0 on success.

    compute-sanitizer --tool memcheck python tests/sanitize_driver.py [cfg] [n] [views]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg=0, n=None, views=1):
    import torch

    from paper_2409_04751_b200 import BackwardOptions, Rasterizer, RenderOptions, synthetic
    from tests._helpers import to_device

    kw = {"n": n} if n else {}
    if cfg >= 3:
        kw["views"] = views
    scene, deg, cams, dls = synthetic.config(cfg, **kw)
    ds = to_device(scene)
    r = Rasterizer(0)
    o = RenderOptions(sh_degree=deg)
    grads = torch.zeros(59 * scene.n, dtype=torch.float32, device="cuda")
    for it in range(2):
        for v, cam in enumerate(cams):
            dl = (torch.from_numpy(dls[v % len(dls)]).cuda() if dls else
                  torch.randn((cam.height, cam.width, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(v)))
            r.forward(ds, cam, o)
            r.backward(ds, cam, dl, BackwardOptions(), grads=grads, accumulate=v > 0)
    torch.cuda.synchronize()
    img, _, _ = r.render_host(scene, cams[0], o)
    assert np.isfinite(img).all() and np.isfinite(grads.cpu().numpy()).all()
    print("sanitize-driver ok")


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
