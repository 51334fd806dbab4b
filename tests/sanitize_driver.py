"""Driver for the checked-build runs (tests/test_checked_gpu.py, or by hand): forward + backward of
one BASELINE config on cuda:0 through the C ABI after a frame of a scene prefix (so the first full
frame grows the buffers and relaunches), twice (the second takes the speculative launch path), once
more with the counters and blend-count flags (the forward's other kernel modes), then a host-buffer render and, for configs 3-4, the native multi-view step. Exits 0 on success;
a failed device check in libfgs_checked.so prints its site and traps, which fails the run.

    FGS_LIB=checked python tests/sanitize_driver.py [cfg] [n] [views] [flags]

The kernel variants are chosen with the library's env overrides (FGS_FWD_PX, FGS_BWD_PX,
FGS_FWD_TMA, ...); `flags` are extra FGS_FLAG_* bits for every frame (e.g. 16 / 32: row / slot
scatter order). (compute-sanitizer would be the tool for this; it is closed on this GPU pool.)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg=0, n=0, views=1, flags=0):
    import torch

    from paper_2409_04751_b200 import BackwardOptions, Rasterizer, RenderOptions, Scene, _lib, synthetic
    from tests._helpers import to_device

    L = _lib.load()
    print("library:", L._name)
    kw = {"n": n} if n else {}
    if cfg >= 3:
        kw["views"] = views
    scene, deg, cams, dls = synthetic.config(cfg, **kw)
    ds = to_device(scene)
    r = Rasterizer(0)
    o = RenderOptions(sh_degree=deg)
    grads = torch.zeros(59 * scene.n, dtype=torch.float32, device="cuda")
    # a prefix of the scene first: the full scene's first frame then overflows the buffers the
    # prefix sized and takes the grow-and-relaunch path
    k = max(1, scene.n // 8)
    pre = Scene(ds.means[:k], ds.rotations[:k], ds.log_scales[:k], ds.opacity_logits[:k], ds.sh[:k], ds.background)
    r.forward(pre, cams[0], o)
    torch.cuda.synchronize()
    dl_dev = []
    for v, cam in enumerate(cams):
        dl_dev.append(torch.from_numpy(dls[v % len(dls)]).cuda() if dls else
                      torch.randn((cam.height, cam.width, 3), device="cuda",
                                  generator=torch.Generator("cuda").manual_seed(v)))
    for it, fl in enumerate((flags, flags, flags | _lib.FGS_FLAG_COUNTERS | _lib.FGS_FLAG_BLEND_COUNT)):
        r.set_flags(fl)
        for v, cam in enumerate(cams):
            r.forward(ds, cam, o)
            r.backward(ds, cam, dl_dev[v], BackwardOptions(), grads=grads, accumulate=v > 0)
        torch.cuda.synchronize()
    r.set_flags(flags)
    img, _, _ = r.render_host(scene, cams[0], o)
    if cfg >= 3:
        g2 = r.fwd_bwd_views(ds, cams, dl_dev, o)
        torch.cuda.synchronize()
        assert np.isfinite(g2.cpu().numpy()).all()
    assert np.isfinite(img).all() and np.isfinite(grads.cpu().numpy()).all()
    print("sanitize-driver ok")


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
