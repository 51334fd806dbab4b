"""Per-tile CTA timeline of the forward and backward blends (FGS_FLAG_COUNTERS, %globaltimer):
how long the heaviest tiles' CTAs run against the whole kernel, i.e. whether the blend is bound
by its slowest tile (a serial chain) rather than by throughput.

    python profiles/tile_tail.py [cfg]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def report(name, span, off):
    span = span.reshape(-1, 2).astype(np.int64)
    ok = span[:, 0] > 0
    t0 = span[ok, 0].min()
    s, e = span[:, 0] - t0, span[:, 1] - t0
    dur = (e - s)[ok]
    total = e[ok].max()
    L = np.diff(off.astype(np.int64))[ok]
    ends = np.sort(e[ok])
    q = lambda f: ends[int(f * (len(ends) - 1))] / 1e3
    print(f"{name}: kernel span {total / 1e3:.1f} us; CTAs done at 50% {q(.5):.1f} 90% {q(.9):.1f} "
          f"99% {q(.99):.1f} 99.9% {q(.999):.1f} us; last CTA start {s[ok].max() / 1e3:.1f} us")
    top = np.argsort(-dur)[:8]
    print("   slowest tiles (us, list length, start us):",
          [(round(dur[i] / 1e3, 1), int(L[i]), round(s[ok][i] / 1e3, 1)) for i in top])
    # duration vs list length
    for lo, hi in ((0, 64), (64, 256), (256, 1024), (1024, 1 << 30)):
        m = (L >= lo) & (L < hi)
        if m.any():
            print(f"   lists [{lo},{hi}): {m.sum()} tiles, mean {dur[m].mean() / 1e3:.1f} us, max {dur[m].max() / 1e3:.1f} us")


def main(cfg=2):
    import torch

    from paper_2409_04751_b200 import BackwardOptions, Rasterizer, RenderOptions, _lib, synthetic
    from tests._helpers import to_device

    sc, deg, cams, dls = synthetic.config(cfg, **({"views": 1} if cfg >= 3 else {}))
    ds = to_device(sc)
    r = Rasterizer(0)
    o = RenderOptions(sh_degree=deg)
    dl = torch.from_numpy(dls[0]).cuda() if dls else torch.randn((cams[0].height, cams[0].width, 3), device="cuda")
    for _ in range(3):
        r.forward(ds, cams[0], o)
        r.backward(ds, cams[0], dl, BackwardOptions())
    r.set_flags(_lib.FGS_FLAG_COUNTERS)
    r.forward(ds, cams[0], o)
    r.backward(ds, cams[0], dl, BackwardOptions())
    torch.cuda.synchronize()
    off = r.debug("offsets")
    c16 = r.debug("counters16", np.uint64).astype(np.float64)
    span = r.debug("tile_span", np.uint64).reshape(-1, 2).astype(np.float64)
    ok = span[:, 0] > 0
    cta_ns = (span[ok, 1] - span[ok, 0]).sum()
    sort_cyc = c16[4] + c16[5]
    print(f"forward sort phase: {sort_cyc / 1.965 / cta_ns * 100:.1f} % of the summed CTA durations "
          f"(short lists {c16[4] / max(sort_cyc, 1) * 100:.0f} %, long lists {int(c16[6])} of {int(c16[7])} tiles)")
    report("forward blend", r.debug("tile_span", np.uint64), off)
    report("backward blend", r.debug("tile_span_bwd", np.uint64), off)
    r.set_flags(0)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
