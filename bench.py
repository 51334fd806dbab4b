"""Benchmark: Fisheye-GS rasterizer on B200 (BASELINE.json metric).

Default workload (N=1): config 2 — 1,000,000 clustered Gaussians, SH degree 3, one
1752x1168 equidistant-fisheye view (the north-star ">= 500 FPS forward" case). A step is one
forward render of that view; `value` is forward FPS (frames/s, whole job = sum over ranks).
Fwd+bwd views/s on the same scene is reported beside it. Multi-GPU: each rank renders its own
replica (camera-partitioned, no collective) -> "scaling": "weak"; `--workload cfg4` runs the
multi-view fwd+bwd step with the NCCL gradient all-reduce.

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the reference
headers compiled against the repo's Eigen shim; falls back to the oracle port) on the host
cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FPS @1752x1168 fwd and fwd+bwd views/s at 1/2/4/8 B200; % HBM/FP32 roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="cfg2", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, ws, rank)
    import torch

    from paper_2409_04751_b200 import BackwardOptions, Rasterizer, RenderOptions, synthetic
    from paper_2409_04751_b200.api import split_grads

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local)
    cfg = int(args.workload[3:])
    scene, deg, cams, dls = synthetic.config(cfg, rank=rank)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    from paper_2409_04751_b200.types import Scene

    ds = Scene(t(scene.means), t(scene.rotations), t(scene.log_scales), t(scene.opacity_logits), t(scene.sh),
               scene.background)
    if cfg == 3:  # views partitioned by camera across ranks
        cams = cams[rank::ws]
    cam = cams[0]
    r = Rasterizer(local)
    stream = torch.cuda.current_stream(dev)
    r.set_stream(stream.cuda_stream)
    opts = RenderOptions(sh_degree=deg)
    image = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=dev)
    dl = t(dls[0]) if dls else torch.randn((cam.height, cam.width, 3), device=dev)
    grads = torch.zeros(59 * scene.n, dtype=torch.float32, device=dev)

    def step_fwd():
        for c in (cams if cfg == 3 else [cam]):
            r.forward(ds, c, opts, image=image)

    def step_fwdbwd():
        views = cams if cfg == 4 else [cam]
        for i, c in enumerate(views):
            r.forward(ds, c, opts, image=image)
            r.backward(ds, c, t(dls[i]) if (cfg == 4 and dls) else dl, BackwardOptions(), grads=grads,
                       accumulate=i > 0)
        if cfg == 4 and dist is not None:
            dist.all_reduce(grads)

    primary = step_fwdbwd if cfg in (1, 4) else step_fwd
    views_per_step = len(cams) if cfg == 3 else (len(cams) if cfg == 4 else 1)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        ms = e0.elapsed_time(e1) / steps
        if dist is not None:
            tm = torch.tensor([ms], device=dev)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            ms = float(tm.item())
        return ms

    with ClockSampler(local) as clk:
        ms = timed(primary, args.steps, args.warmup)
    # secondary: fwd+bwd on the same workload (single view)
    ms_fb = timed(lambda: (r.forward(ds, cam, opts, image=image),
                           r.backward(ds, cam, dl, BackwardOptions(), grads=grads)), max(3, args.steps // 2), 2)
    _, st = r.forward(ds, cam, opts, image=image, want_stats=True)
    torch.cuda.synchronize()

    value = ws * views_per_step * 1000.0 / ms
    res = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "views/s" if cfg in (1, 3, 4) else "FPS",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded numpy, BASELINE.json config %d)" % cfg,
        "config": {"workload": args.workload, "gaussians": scene.n, "sh_degree": deg, "width": cam.width,
                   "height": cam.height, "views_per_rank": views_per_step, "parallelism": f"camera-partitioned x{ws}",
                   "l2": "inputs (%.0f MB of Gaussian parameters per step) exceed the 126 MB L2" % (scene.n * 236 / 1e6)},
        "fwd_bwd_views_per_s": round(ws * 1000.0 / ms_fb, 2),
        "stage_ms": {"preprocess": st.preprocess_ms, "binning": st.binning_ms, "sort": st.sort_ms,
                     "raster": st.raster_ms},
        "num_intersections": st.num_intersections,
        "num_splats": st.num_splats,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(res))
    if dist is not None:
        dist.destroy_process_group()


def run_reference(args, ws, rank):
    if rank != 0:
        return
    print(json.dumps({"impl": "reference", "unavailable": "not wired yet"}))


if __name__ == "__main__":
    main()
