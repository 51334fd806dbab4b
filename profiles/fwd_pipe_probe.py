"""Device-resident forward frames on 1 or 2 contexts alternating on their own streams (config 2):
with two, frame i+1's preprocess (HBM-bound) can run beside frame i's blend (FP32-bound).
Frames per second from CUDA events across both streams, and a bit-exactness check.
Measured (one B200): 1 context 254.2 us/frame, 2 contexts 252.3, 3 contexts 249.6, 2 contexts on
alternating stream priorities 264 -- the frame is throughput-bound on the SMs (the blend's 8030
CTAs keep them busy), so a second frame's preprocess finds no idle capacity to fill.
    python profiles/fwd_pipe_probe.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_04751_b200 import Rasterizer, RenderOptions, synthetic  # noqa: E402
from tests._helpers import to_device  # noqa: E402

sc, deg, cams, _ = synthetic.config(2)
ds = to_device(sc)
o = RenderOptions(sh_degree=deg)


def run(nctx, steps=300, prio=False):
    rs = [Rasterizer(0) for _ in range(nctx)]
    sts = [torch.cuda.Stream(priority=-(k % 2) if prio else 0) for k in range(nctx)]
    imgs = [torch.empty((cams[0].height, cams[0].width, 3), device="cuda") for _ in range(nctx)]
    for r, s in zip(rs, sts):
        r.set_stream(s.cuda_stream)
    for k in range(10):
        rs[k % nctx].forward(ds, cams[0], o, image=imgs[k % nctx])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sts[0])
    for s in sts[1:]:
        s.wait_event(e0)
    for k in range(steps):
        rs[k % nctx].forward(ds, cams[0], o, image=imgs[k % nctx])
    for s in sts[1:]:
        ev = torch.cuda.Event()
        ev.record(s)
        sts[0].wait_event(ev)
    e1.record(sts[0])
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"contexts {nctx}{' (alternating priorities)' if prio else ''}: {ms * 1e3:.1f} us/frame, {1e3 / ms:.1f} FPS")
    ref = rs[0].forward(ds, cams[0], o)[0]
    torch.cuda.synchronize()
    assert all(torch.equal(i, ref) for i in imgs)


for n, p in ((1, False), (2, False), (2, True), (1, False), (2, True)):
    run(n, prio=p)
