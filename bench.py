"""Benchmark: B200 Fisheye-GS rasterizer (BASELINE.json metric).

Default workload (N=1): BASELINE.json config 2 — 1,000,000 clustered Gaussians, SH degree 3,
one 1752x1168 equidistant-fisheye view (the north-star ">= 500 FPS forward" case). A step is
one forward render of that view with the Gaussians resident in HBM; `value` is forward FPS
(whole job: summed over ranks). Fwd+bwd views/s of the same view is reported beside it.
`e2e` is the same metric through the reference-facing host call (fgs_render_host: pinned host
scene in, host image out, H2D/D2H copies inside the timed region).

Multi-GPU (torchrun, one rank per GPU): the path shards by camera with the Gaussians replicated;
for the default workload every rank renders its own replica view, no collective ("weak").
`--workload cfg3` = batched forward of 64 views partitioned over ranks; `--workload cfg4` = 8
views/GPU fwd+bwd with the one NCCL all-reduce of the 59*N gradient buffer.

`--impl reference` times the reference's own CPU implementation on the host cores: the
reference headers compiled against the repo's Eigen shim (oracle/_ref), else the oracle port.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FPS @1752x1168 fwd and fwd+bwd views/s at 1/2/4/8 B200; % HBM/FP32 roofline"
FWD_ONLY = {0: True, 1: False, 2: True, 3: True, 4: False}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="cfg2", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu):
        self.gpu, self.samples, self._stop, self._t = gpu, [], threading.Event(), None

    def sample(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
            if out.strip():
                self.samples.append([x.strip() for x in out.strip().split(",")])
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else None
        sm = [num(s[0]) for s in self.samples if num(s[0])]
        mx = [num(s[1]) for s in self.samples if num(s[1])]
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def workload(cfg, rank, ws):
    from paper_2409_04751_b200 import multiview, synthetic

    scene, deg, cams, dls = synthetic.config(cfg, rank=rank)
    if cfg == 3:
        mine = multiview.partition_views(len(cams), ws, rank)
        cams = [cams[v] for v in mine]
    return scene, deg, cams, dls


def stage_work(cfg, scene, deg, st, counters):
    """Algorithmic work per launch of each stage, SURVEY.md §8(d)'s per-unit figures:
    K1 preprocess N*B_in + 48N bytes; K2 duplicate+sort+ranges 8N + 116*I bytes; K3 blend
    11*E_eval + 13*E_contrib flop; K4a 11*E_eval + 60*E_contrib flop; K4b 472N + 48*N_v bytes."""
    n, nv, I = scene.n, st["num_splats"], st["num_intersections"]
    b_in = 236 if deg == 3 else 56
    e_eval, e_con = counters
    return {
        "preprocess": ("hbm", n * b_in + 48 * n),
        "binning+sort": ("hbm", 8 * n + 116 * I),
        "raster": ("fp32", 11 * e_eval + 13 * e_con),
        "raster_backward": ("fp32", 11 * e_eval + 60 * e_con),
        "preprocess_backward": ("hbm", 472 * n + 48 * nv),
    }


def run_ours(args, ws, rank, local):
    import torch

    from paper_2409_04751_b200 import BackwardOptions, Rasterizer, RenderOptions, _lib, multiview
    from paper_2409_04751_b200.types import Scene

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local)
    cfg = int(args.workload[3:])
    scene, deg, cams, dls = workload(cfg, rank, ws)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ds = Scene(to(scene.means), to(scene.rotations), to(scene.log_scales), to(scene.opacity_logits), to(scene.sh),
               scene.background)
    cam = cams[0]
    r = Rasterizer(local)
    stream = torch.cuda.current_stream(dev)
    r.set_stream(stream.cuda_stream)
    ropt = RenderOptions(sh_degree=deg)
    bopt = BackwardOptions()
    image = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=dev)
    dl_dev = [to(d) for d in dls] if dls else [torch.randn((cam.height, cam.width, 3), device=dev)]
    grads = torch.zeros(59 * scene.n, dtype=torch.float32, device=dev)

    def fwd_views():
        multiview.forward_views(cams, lambda c: r.forward(ds, c, ropt, image=image))

    # config 4 over several GPUs: the library's own NCCL communicator (csrc/comm.cu), the id shared
    # over the torch.distributed group; the all-reduce overlaps the last view's preprocess backward
    comm = multiview.Communicator.from_process_group(r) if (dist is not None and cfg == 4) else None

    def fwd_bwd_views(views):
        # the native rank step: forward + accumulating backward of every view (+ the all-reduce)
        r.fwd_bwd_views(ds, [cams[i] for i in views], [dl_dev[i % len(dl_dev)] for i in views], ropt, bopt,
                        grads=grads, comm=comm)

    views = list(range(len(cams)))
    primary = fwd_views if FWD_ONLY[cfg] else (lambda: fwd_bwd_views(views))
    views_per_step = len(cams) if cfg in (3, 4) else 1

    # Per-stage CUDA events (FGS_FLAG_TIMING) are recorded on every 8th step of a timed loop:
    # timing events between kernels keep the GPU from starting a kernel while the previous
    # one drains (~17 us per forward at config 2), so the other steps run unperturbed.
    stage_every = 8

    scene_bytes = scene.n * (236 if deg == 3 else 56)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if scene_bytes < 126e6 else None

    def timed(fn, steps, warmup, sampler=None, finish=None, allow_flush=True):
        r.set_flags(0)
        for _ in range(warmup):
            fn()
        if finish:
            finish()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        r.timing(reset=True)
        if sampler:
            sampler.sample()
        use_flush = flush is not None and allow_flush
        if not use_flush:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(steps):
                r.set_flags(_lib.FGS_FLAG_TIMING if i % stage_every == 0 else 0)
                fn()
            if finish:
                finish()  # (the last asynchronous frame's read-back, inside the timed region)
            e1.record(stream)
        else:
            # scene smaller than the L2: L2 flushed (a 256 MB write) before every step, each step
            # timed by its own event pair so the flush is not counted
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for i in range(steps):
                flush.zero_()
                r.set_flags(_lib.FGS_FLAG_TIMING if i % stage_every == 0 else 0)
                ev[i][0].record(stream)
                fn()
                if finish:
                    finish()
                ev[i][1].record(stream)
        r.set_flags(0)
        torch.cuda.synchronize()
        if sampler:
            sampler.sample()
        if dist is not None:
            dist.barrier()
        ms = (e0.elapsed_time(e1) if not use_flush else sum(a.elapsed_time(b) for a, b in ev)) / steps
        if dist is not None:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, r.timing(reset=True)

    clk = ClockSampler(local)
    with clk:
        ms, tim = timed(primary, args.steps, args.warmup, clk)
    launches = tim["launches"]
    # fwd+bwd of the first view (secondary number for forward-only workloads)
    ms_fb, tim_fb = timed(lambda: fwd_bwd_views([0]), max(5, args.steps // 4), 3)
    r.set_flags(0)

    # work counters and stats of the measured view (instrumented run, outside the timed region)
    r.set_flags(_lib.FGS_FLAG_COUNTERS)
    _, st = r.forward(ds, cam, ropt, image=image, want_stats=True)
    r.backward(ds, cam, dl_dev[0], bopt, grads=grads)
    vv = r.debug("variants").tolist()
    variants = {"fwd_pixels_per_lane": vv[0], "bwd_pixels_per_lane": vv[1], "k4b_ctas_per_sm": vv[2],
                "longest_tile_list": vv[3], "binning_scatter": "tile-row lists" if vv[4] else ("CTA-local slots" if vv[5] else "source-order slots"),
                "rule": "deterministic from frame statistics (fgs_api.cu rule_*)"}
    counters_all = r.debug("counters", np.uint64).tolist()
    counters = counters_all[:2]
    r.set_flags(0)
    stn = {"num_splats": st.num_splats, "num_intersections": st.num_intersections}
    work = stage_work(cfg, scene, deg, stn, counters)

    peaks, peak_src = measured_peaks()
    fp32_peak = r.fp32_peak()  # non-FMA fp32 op/s, measured on this device now
    stage_ms = {}
    calls_f, calls_b = max(1, tim["forward_calls"]), max(1, tim["backward_calls"])
    for k, v in tim["ms"].items():
        c = calls_f if k in ("preprocess", "binning", "sort", "raster") else calls_b
        if v > 0:
            stage_ms[k] = v / c
    for k, v in tim_fb["ms"].items():
        if k not in stage_ms and v > 0:
            stage_ms[k] = v / max(1, tim_fb["backward_calls"])
    if "binning" in stage_ms or "sort" in stage_ms:
        stage_ms["binning+sort"] = stage_ms.get("binning", 0.0) + stage_ms.get("sort", 0.0)
    rooflines = {}
    for k, t_ms in stage_ms.items():
        if k not in work:
            continue
        bound, amount = work[k]
        if bound == "hbm":
            ach = amount / (t_ms * 1e-3) / 1e9
            rooflines[k] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                            "frac": round(ach / peaks["hbm_gbs"], 4), "ms": round(t_ms, 4), "work": int(amount)}
        else:
            ach = amount / (t_ms * 1e-3) / 1e12
            pk = fp32_peak / 1e12
            rooflines[k] = {"bound": "fp32", "achieved": round(ach, 3), "peak": round(pk, 2), "unit": "TFLOP/s",
                            "frac": round(ach / pk, 4), "ms": round(t_ms, 4), "work": int(amount)}
    primary_stages = ["preprocess", "binning+sort", "raster"] + ([] if FWD_ONLY[cfg] else
                                                                    ["raster_backward", "preprocess_backward"])
    def dominant(stages):
        dom = max((k for k in stages if k in rooflines), key=lambda k: rooflines[k]["ms"])
        roof = dict(rooflines[dom])
        roof["kernel"] = dom
        roof["traffic"] = load_traffic(dom)
        roof["peak_source"] = ("fp32 probe kernel on this device (FMUL+FADD, non-FMA ops)" if roof["bound"] == "fp32"
                               else f"MEASURED_PEAKS.json hbm_gbs ({peak_src})")
        return roof

    # (K1's figure counts every Gaussian's 192-byte SH row; K1 reads the rows of Gaussians that
    # project near the image only, and is issue / latency-bound, not HBM-bound: DESIGN.md §8)
    if "preprocess" in rooflines:
        rooflines["preprocess"]["note"] = ("issue/latency-bound (ncu: ~76% issue, ~155 MB DRAM per launch at "
                                           "config 2); the algorithmic bytes count all SH rows")
    roof = dominant(primary_stages)
    # the metric's second half (fwd+bwd views/s): dominant stage of forward + backward
    roof_fb = dominant(["preprocess", "binning+sort", "raster", "raster_backward", "preprocess_backward"])

    # e2e through the reference-facing host call (pinned host buffers, copies in the timed region)
    e2e = None
    if cfg in (0, 1, 2):
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        hs = Scene(pin(scene.means), pin(scene.rotations), pin(scene.log_scales), pin(scene.opacity_logits),
                   pin(scene.sh), scene.background)
        himg = torch.empty((cam.height, cam.width, 3), dtype=torch.float32).pin_memory().numpy()
        himg2 = [himg, torch.empty((cam.height, cam.width, 3), dtype=torch.float32).pin_memory().numpy()]
        hdl = pin(dls[0]) if dls else None
        hgr = torch.zeros(59 * scene.n, dtype=torch.float32).pin_memory().numpy()
        finish = None
        if FWD_ONLY[cfg]:
            # a stream of frames through the pipelined host call: each frame reads its scene over
            # PCIe and reads its image back, the read-back overlapping the next frame's scene reads
            k = [0]

            def step():
                r.render_host_async(hs, cam, ropt, radii=None, image=himg2[k[0] & 1], want_stats=False)
                k[0] += 1
            finish = r.wait
        else:
            # forward + backward frames through the pipelined host calls: each frame's image and
            # gradient read-backs overlap the next frame's scene reads and dL/dimage upload
            hgr2 = [hgr, torch.zeros(59 * scene.n, dtype=torch.float32).pin_memory().numpy()]
            k = [0]

            def step():
                r.render_host_async(hs, cam, ropt, radii=None, image=himg2[k[0] & 1], want_stats=False)
                r.backward_host_async(hs, cam, hdl, bopt, grads=hgr2[k[0] & 1])
                k[0] += 1
            finish = r.wait
        e_steps = max(3, min(args.steps, 20))
        # (no L2 flush: every step streams its inputs from host memory)
        ms_e2e, _ = timed(step, e_steps, 2, finish=finish, allow_flush=False)
        # bytes actually moved over PCIe per step (pinned scene arrays are read in place by K1 /
        # K4b, only what they touch): measured by the library on the last step
        if FWD_ONLY[cfg]:
            h2d, d2h = r.last_transfer()["h2d"], r.last_transfer()["d2h"]
        else:
            r.render_host(hs, cam, ropt, radii=None, image=himg, want_stats=False)
            fwd_t = r.last_transfer()
            r.backward_host(hs, cam, hdl, bopt, grads=hgr)
            bwd_t = r.last_transfer()
            h2d, d2h = fwd_t["h2d"] + bwd_t["h2d"], fwd_t["d2h"] + bwd_t["d2h"]
        e2e = {"value": round(ws * 1000.0 / ms_e2e, 2), "unit": "FPS" if FWD_ONLY[cfg] else "views/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms_e2e, 3),
               "path": ("fgs_render_host_async (pipelined frames: each frame's image read-back overlaps "
                        "the next frame's zero-copy scene reads)") if FWD_ONLY[cfg] else
                       ("fgs_render_host_async + fgs_backward_host_async (pipelined frames: image and gradient "
                        "read-backs overlap the next frame's scene reads and dL/dimage upload)")}

    cpu = cpu_fb = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, scene, deg, cams, dls, args.cpu_seconds)
        # the reference backward (gradients.hpp:207-267) timed too: forward+backward views/s
        cpu_fb = cpu if not FWD_ONLY[cfg] else cpu_baseline(cfg, scene, deg, cams, dls, args.cpu_seconds,
                                                            fwd_only=False)

    value = ws * views_per_step * 1000.0 / ms
    unit = "FPS" if cfg in (0, 2) else "views/s"
    res = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": unit,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": f"synthetic: seeded numpy draws of BASELINE.json config {cfg} (no dataset)",
        "config": bench_config(args, cfg, scene, deg, cam, views_per_step, ws),
        "e2e": e2e,
        "roofline": roof,
        "roofline_fwd_bwd": roof_fb,
        "cpu_baseline": cpu,
        "cpu_baseline_fwd_bwd": cpu_fb,
        "variants": variants,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "fwd_bwd_views_per_s": round(ws * 1000.0 / ms_fb, 2),
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "stage_roofline": rooflines,
        "num_intersections": st.num_intersections,
        "num_splats": st.num_splats,
        "e_eval": int(counters[0]),
        "e_contrib": int(counters[1]),
        "blend_pixel_evals_after_culling": int(counters_all[2]),
        "fp32_peak_tops": round(fp32_peak / 1e12, 2),
    }
    if rank == 0:
        print(json.dumps(res))
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


def views_per_rank(cfg, n_views, ws):
    from paper_2409_04751_b200 import multiview

    if cfg == 3:
        return len(multiview.partition_views(n_views, ws, 0))
    return n_views if cfg == 4 else 1


def bench_config(args, cfg, scene, deg, cam, views_per_step, ws):
    """The workload description both arms print (identical dicts)."""
    sb = scene.n * (236 if deg == 3 else 56)
    return {"workload": args.workload, "gaussians": scene.n, "sh_degree": deg, "width": cam.width,
            "height": cam.height, "views_per_rank": views_per_step,
            "step": "forward" if FWD_ONLY[cfg] else "forward+backward",
            "parallelism": f"camera-partitioned x{ws}" + (", NCCL all-reduce of 59N grads" if cfg == 4 else ""),
            "l2": ("no flush: the %.0f MB of Gaussian parameters read per step exceed the 126 MB L2" % (sb / 1e6)
                   if sb >= 126e6 else
                   "L2 flushed (256 MB write) before every timed step, outside its event pair: the %.1f MB scene "
                   "fits the 126 MB L2" % (sb / 1e6))}


def load_traffic(kernel):
    """dram bytes read+write per launch of `kernel` from the committed ncu capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            v = json.load(f).get(kernel)
            return v if v is None else int(v)
    except Exception:
        return None


def _cpu_frame(impl, scene, deg, cam, dl, fwd_only, threads):
    import oracle

    kw = dict(impl="ref") if impl == "reference" else dict(mode=oracle.MODE_LIBM)
    res = oracle.render(scene, cam, sh_degree=deg, threads=threads, **kw)
    if not fwd_only:
        if impl == "reference":
            oracle.backward(res, scene.n, dl, threads=threads)
        else:
            oracle.backward(res, scene.n, dl, threads=threads, full_sh=False, mode=oracle.MODE_LIBM)
    res.close()


def cpu_impl():
    import oracle

    oracle.build()
    return "reference" if oracle.ref_available() else "port"


def cpu_baseline(cfg, scene, deg, cams, dls, budget_s, fwd_only=None):
    """The reference's CPU path on this host's cores, one bounded sample (~budget_s of work).
    fwd_only=False times forward + backward (the reference's backward needs dL/dpixel: the
    config's own, or a seeded N(0, 1) image for the forward-only configs)."""
    impl = cpu_impl()
    threads = os.cpu_count() or 1
    fwd_only = FWD_ONLY[cfg] if fwd_only is None else fwd_only
    if not fwd_only and not dls:
        dls = [np.random.default_rng(7).standard_normal((cams[0].height, cams[0].width, 3)).astype(np.float32)]
    dl = dls[0] if dls else None
    t0 = time.perf_counter()
    _cpu_frame(impl, scene, deg, cams[0], dl, fwd_only, threads)  # warm-up (page-in, thread spawn)
    first = time.perf_counter() - t0
    frames, times = 0, []
    while frames < 1 or (sum(times) < budget_s and frames < 50):
        c = cams[frames % len(cams)]
        t = time.perf_counter()
        _cpu_frame(impl, scene, deg, c, dls[frames % len(dls)] if dls else None, fwd_only, threads)
        times.append(time.perf_counter() - t)
        frames += 1
        if first > budget_s:
            break
    v = frames / sum(times)
    return {"value": round(v, 4), "unit": "FPS" if fwd_only else "views/s", "cores": threads,
            "kind": impl, "sample": f"{frames} full {'forward' if fwd_only else 'forward+backward'} view(s) of the "
                                    f"same workload, fp32, {threads} threads (median {np.median(times):.2f} s/view)"}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cfg = int(args.workload[3:])
    scene, deg, cams, dls = workload(cfg, 0, 1)
    impl = cpu_impl()
    threads = os.cpu_count() or 1
    fwd_only = FWD_ONLY[cfg]
    warm, t_w = 0, time.perf_counter()
    for _ in range(args.warmup):  # all W warm-up steps unless they exceed a minute
        _cpu_frame(impl, scene, deg, cams[0], dls[0] if dls else None, fwd_only, threads)
        warm += 1
        if time.perf_counter() - t_w > 60.0:
            break
    times, steps = [], 0
    t_start = time.perf_counter()
    for i in range(args.steps):
        t = time.perf_counter()
        _cpu_frame(impl, scene, deg, cams[i % len(cams)], dls[i % len(dls)] if dls else None, fwd_only, threads)
        times.append(time.perf_counter() - t)
        steps += 1
        if time.perf_counter() - t_start > 150.0:  # keep the arm within a few minutes
            break
    ms = 1000.0 * sum(times) / steps
    v = round(1000.0 / ms, 4)
    unit = "FPS" if fwd_only and cfg in (0, 2) else "views/s"
    sample = (f"{steps} of {args.steps} requested steps (150 s cap), each one full "
              f"{'forward' if fwd_only else 'forward+backward'} view (views/s is per view); {threads} threads")
    res = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": unit,
        "n_gpus": ws,
        "steps": steps,
        "warmup": warm,
        "ms_per_step": round(ms, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": f"synthetic: seeded numpy draws of BASELINE.json config {cfg} (no dataset)",
        "config": bench_config(args, cfg, scene, deg, cams[0], views_per_rank(cfg, len(cams), ws), ws),
        "cpu_baseline": {"kind": impl, "cores": threads, "sample": sample, "value": v, "unit": unit},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(res))


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, ws, rank)
    return run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
