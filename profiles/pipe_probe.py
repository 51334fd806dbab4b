"""Pipelined host-buffer frames (fgs_render_host_async) on 1, 2 or 3 contexts alternating on
their own streams, config 2: frames per second and a bit-exactness check. Measured (one B200):
1 context 2.287 ms/frame (437 FPS), 2 contexts 2.285, 3 contexts 2.282 -- a call returns only
once its frame's binning scalars are known, so a second context cannot start the next frame's
PCIe-bound preprocess any earlier than the first context's queue does.
    python profiles/pipe_probe.py
"""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2409_04751_b200 import Rasterizer, RenderOptions, Scene, synthetic
sc, deg, cams, _ = synthetic.config(2)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory().numpy()
hs = Scene(pin(sc.means), pin(sc.rotations), pin(sc.log_scales), pin(sc.opacity_logits), pin(sc.sh), sc.background)
o = RenderOptions(sh_degree=deg)
imgs = [torch.empty((cams[0].height, cams[0].width, 3), dtype=torch.float32).pin_memory().numpy() for _ in range(4)]
def run(nctx, steps=40):
    rs = [Rasterizer(0) for _ in range(nctx)]
    sts = [torch.cuda.Stream() for _ in range(nctx)]
    for r, s in zip(rs, sts): r.set_stream(s.cuda_stream)
    for k in range(6): rs[k % nctx].render_host_async(hs, cams[0], o, image=imgs[k % 4], want_stats=False)
    for r in rs: r.wait()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps): rs[k % nctx].render_host_async(hs, cams[0], o, image=imgs[k % 4], want_stats=False)
    for r in rs: r.wait()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    print(f"contexts {nctx}: {dt*1e3:.3f} ms/frame, {1/dt:.1f} FPS")
    ref = Rasterizer(0).render_host(hs, cams[0], o)[0]
    assert all(i.tobytes() == ref.tobytes() for i in imgs), "mismatch"
for n in (1, 2, 3):
    run(n)
