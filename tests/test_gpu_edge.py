"""GPU edge cases and API behaviour through the C ABI (reference error semantics, empty and
all-culled scenes, ragged image sizes, determinism, multi-view accumulation, host path)."""
import math

import numpy as np
import pytest

from tests._helpers import GROUPS, rel_l2, small_fisheye, to_device
from tests.golden.make_golden import spherical_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rast():
    import torch

    assert torch.cuda.is_available()
    from paper_2409_04751_b200 import Rasterizer

    return Rasterizer(0)


def fwd(rast, scene, cam, deg=3):
    import torch
    from paper_2409_04751_b200 import RenderOptions

    img, st = rast.forward(to_device(scene), cam, RenderOptions(sh_degree=deg, background=scene.background),
                           want_stats=True)
    torch.cuda.synchronize()
    return img.cpu().numpy(), st


def test_empty_scene_is_background(rast):  # test_splatting.cpp:191-199
    from paper_2409_04751_b200 import Scene

    sc = Scene(np.zeros((0, 3), np.float32), np.zeros((0, 4), np.float32), np.zeros((0, 3), np.float32),
               np.zeros(0, np.float32), np.zeros((0, 48), np.float32), np.array([0.3, 0.5, 0.7], np.float32))
    img, st = fwd(rast, sc, small_fisheye(48, 32))
    assert st.num_intersections == 0
    assert (img == np.array([0.3, 0.5, 0.7], np.float32)).all()


def test_all_culled_scene(rast):
    sc = spherical_scene(100, 2)
    sc.means[:] = np.array([0, 0, -5.0], np.float32)  # on the backward axis
    img, st = fwd(rast, sc, small_fisheye())
    assert st.num_intersections == 0 and st.num_splats == 0 and st.num_culled == 100
    assert (img == sc.background).all()


def test_degenerate_quaternion_raises(rast):  # model.hpp:98
    from paper_2409_04751_b200 import InvalidArgument

    sc = spherical_scene(200, 3)
    cam = small_fisheye()
    import oracle

    res = oracle.render(sc, cam)
    i = int(res.get("source")[0])
    sc.rotations[i] = 0
    with pytest.raises(InvalidArgument, match="degenerate rotation"):
        fwd(rast, sc, cam)


def test_context_recovers_after_errors_and_empty_frames(oracle_mod):
    """A context's per-frame device state (the double-buffered scalars, the speculative launch
    against last frame's capacity, the launch-variant timing) survives a failed frame and an
    empty scene: every later frame matches the oracle."""
    import torch
    from paper_2409_04751_b200 import InvalidArgument, Rasterizer, RenderOptions, Scene

    r = Rasterizer(0)
    good = spherical_scene(2500, 7)
    bad = spherical_scene(2500, 7)
    bad.rotations[3] = 0
    empty = Scene(good.means[:0], good.rotations[:0], good.log_scales[:0], good.opacity_logits[:0], good.sh[:0],
                  good.background)
    cam = small_fisheye(320, 240)
    ref = oracle_mod.render(good, cam, sh_degree=3)
    for sc in (good, bad, good, empty, good, bad, bad, good, good):
        if sc is bad:
            with pytest.raises(InvalidArgument):
                r.forward(to_device(sc), cam, RenderOptions(sh_degree=3, background=sc.background))
            continue
        img, st = r.forward(to_device(sc), cam, RenderOptions(sh_degree=3, background=sc.background),
                            want_stats=True)
        torch.cuda.synchronize()
        if sc is empty:
            assert st.num_intersections == 0
            continue
        assert st.num_intersections == ref.num_intersections
        np.testing.assert_array_equal(r.debug("offsets"), ref.get("offsets"))
        assert np.abs(img.cpu().numpy().astype(np.float64) - ref.image).max() <= 1e-3


def test_backward_rejects_mismatched_context(rast):  # test_gradients.cpp:287-299
    import torch
    from paper_2409_04751_b200 import InvalidArgument

    sc = spherical_scene(300, 4)
    cam = small_fisheye()
    fwd(rast, sc, cam)
    dl = torch.zeros((cam.height, cam.width, 3), device="cuda")
    with pytest.raises(InvalidArgument, match="different scene"):
        rast.backward(to_device(sc.subset(slice(0, 299))), cam, dl)
    cam2 = small_fisheye()
    cam2.fx += 1.0
    with pytest.raises(InvalidArgument, match="different camera"):
        rast.backward(to_device(sc), cam2, dl)
    with pytest.raises(InvalidArgument, match="shape"):
        rast.backward(to_device(sc), cam, torch.zeros((2, 2, 3), device="cuda"))


@pytest.mark.parametrize("wh", [(256, 256), (100, 37), (17, 16), (1752, 1168), (2600, 2100)])
def test_ragged_sizes_and_tile_edges(rast, oracle_mod, wh):
    """W, H multiples of 16 exercise the zero-tile splat (mx - r == W passes the cull,
    splatting.hpp:107-108 / 211-214); odd sizes exercise partial edge tiles."""
    # (2600 x 2100: 163 x 132 = 21516 tiles, past the binning scatter's 16384-tile shared
    # counters, takes the global-atomic scatter)
    w, h = wh
    sc = spherical_scene(3000, 5)
    cam = small_fisheye(w, h)
    img, st = fwd(rast, sc, cam)
    res = oracle_mod.render(sc, cam, sh_degree=3)
    assert st.num_intersections == res.num_intersections and st.num_splats == res.num_splats
    np.testing.assert_array_equal(rast.debug("offsets"), res.get("offsets"))
    np.testing.assert_array_equal(rast.debug("sorted_gauss"), res.get("source")[res.get("refs")])
    assert np.abs(img.astype(np.float64) - res.image).max() <= 1e-3


def test_forward_and_backward_are_deterministic(rast):
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions

    from paper_2409_04751_b200 import synthetic

    sc, deg, cams, dls = synthetic.config(2, n=60000)
    ds = to_device(sc)
    dl = torch.from_numpy(dls[0]).cuda()
    outs = []
    for _ in range(3):
        img, _ = rast.forward(ds, cams[0], RenderOptions(sh_degree=deg))
        g = rast.backward(ds, cams[0], dl, BackwardOptions())
        torch.cuda.synchronize()
        outs.append((img.cpu().numpy().tobytes(), g.cpu().numpy().tobytes()))
    assert outs[0] == outs[1] == outs[2]


def test_forward_independent_of_pixels_per_lane(rast):
    """A fresh context's frames: the work decomposition follows the last frame's statistics
    (deterministic rules), and every frame's image is the same bits."""
    import torch
    from paper_2409_04751_b200 import Rasterizer, RenderOptions, synthetic

    r = Rasterizer(0)  # fresh context: starts tuning
    sc, deg, cams, _ = synthetic.config(1, n=40000)
    ds = to_device(sc)
    imgs = set()
    for _ in range(16):
        img, _ = r.forward(ds, cams[0], RenderOptions(sh_degree=deg))
        torch.cuda.synchronize()
        imgs.add(img.cpu().numpy().tobytes())
    assert len(imgs) == 1


def test_multiview_accumulate_equals_sum(rast):
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, synthetic

    sc, deg, cams, dls = synthetic.config(4, n=20000, views=3)
    ds = to_device(sc)
    acc = torch.zeros(59 * sc.n, device="cuda")
    singles = []
    for i, (c, d) in enumerate(zip(cams, dls)):
        rast.forward(ds, c, RenderOptions(sh_degree=deg))
        dl = torch.from_numpy(d).cuda()
        rast.backward(ds, c, dl, BackwardOptions(), grads=acc, accumulate=i > 0)
        rast.forward(ds, c, RenderOptions(sh_degree=deg))
        singles.append(rast.backward(ds, c, dl, BackwardOptions()).double())
    torch.cuda.synchronize()
    ref = sum(singles)
    assert (torch.linalg.norm(acc.double() - ref) / torch.linalg.norm(ref)).item() < 1e-6


def test_host_path_equals_device_path(rast):
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, backward, render, synthetic
    from paper_2409_04751_b200.api import grads_as_rows

    sc, deg, cams, dls = synthetic.config(1, n=8000)
    res = render(sc, cams[0], RenderOptions(sh_degree=deg), rasterizer=rast)
    g_host = backward(sc, cams[0], res, dls[0], BackwardOptions())
    ds = to_device(sc)
    img, _ = rast.forward(ds, cams[0], RenderOptions(sh_degree=deg))
    g_dev = rast.backward(ds, cams[0], torch.from_numpy(dls[0]).cuda(), BackwardOptions())
    torch.cuda.synchronize()
    assert res.image.tobytes() == img.cpu().numpy().tobytes()
    np.testing.assert_array_equal(g_host["mean"], grads_as_rows(g_dev, sc.n)[:, 0:3])
    assert (res.radii > 0).sum() == res.stats.num_splats


def test_view_dir_gradient_matches_oracle(rast, oracle_mod):
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, grads_as_rows, synthetic

    sc, deg, cams, dls = synthetic.config(4, n=20000, views=1)
    ds = to_device(sc)
    rast.forward(ds, cams[0], RenderOptions(sh_degree=deg))
    g = rast.backward(ds, cams[0], torch.from_numpy(dls[0]).cuda(), BackwardOptions(sh_view_dir_grad=True))
    torch.cuda.synchronize()
    res = oracle_mod.render(sc, cams[0], sh_degree=deg)
    ref, _ = oracle_mod.backward(res, sc.n, dls[0], sh_view_dir_grad=True)
    got = grads_as_rows(g, sc.n)
    for k in ("mean", "rotation", "log_scale", "opacity", "sh_dc", "sh_rest"):
        assert rel_l2(got[:, GROUPS[k]], ref[:, GROUPS[k]]) <= 1e-3, k


def test_counters_match_oracle(rast, oracle_mod):
    """E_eval / E_contrib (the blend's work counters) match the oracle."""
    from paper_2409_04751_b200 import _lib, synthetic

    sc, deg, cams, _ = synthetic.config(0)
    rast.set_flags(_lib.FGS_FLAG_COUNTERS)
    try:
        fwd(rast, sc, cams[0], deg)
        ev, ec, warp_iters, _ = rast.debug("counters", np.uint64)
    finally:
        rast.set_flags(0)
    st = oracle_mod.render(sc, cams[0], sh_degree=deg).stats()
    assert int(ec) == int(st["e_contrib"])
    assert int(ev) == int(st["e_eval"])
    assert 0 < int(warp_iters) <= 2 * int(ev)  # pixel evaluations actually done after culling


def test_cpp_wrapper_example():
    """The C++ host side over the C ABI (include/fgs.hpp) renders, back-propagates and maps the
    reference's std::invalid_argument behaviour."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "tools", "fgs_render_example")
    if not os.path.exists(exe):
        from paper_2409_04751_b200.build import build_example

        build_example()
    out = subprocess.run([exe, "20000", "512", "384"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    kv = dict(tok.split("=") for tok in out.stdout.split() if "=" in tok)
    assert int(kv["intersections"]) > 0 and int(kv["splats"]) > 0
    assert float(kv["image_mean"]) > 0 and float(kv["grad_mean_l1"]) > 0
    assert kv["error_check"] == "ok"


def test_backward_unaligned_gradient_fields(rast, oracle_mod):
    """N not a multiple of 4: the flat 59N gradient buffer's rotation and SH fields are not
    16-byte aligned, so K4b takes its scalar-store path."""
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, grads_as_rows

    sc = spherical_scene(2999, 7)
    cam = small_fisheye(256, 192)
    rast.forward(to_device(sc), cam, RenderOptions(sh_degree=3, background=sc.background))
    dl = np.random.default_rng(3).standard_normal((cam.height, cam.width, 3)).astype(np.float32)
    g = rast.backward(to_device(sc), cam, torch.from_numpy(dl).cuda(), BackwardOptions())
    torch.cuda.synchronize()
    res = oracle_mod.render(sc, cam, sh_degree=3)
    ref, _ = oracle_mod.backward(res, sc.n, dl)
    got = grads_as_rows(g, sc.n)
    for k in ("mean", "rotation", "log_scale", "opacity", "sh_dc", "sh_rest"):
        assert rel_l2(got[:, GROUPS[k]], ref[:, GROUPS[k]]) <= 1e-3, k


@pytest.mark.parametrize("n_distinct,min_len,max_len", [(6000, 2 * 4096, None), (1500, 2049, 4096),
                                                        (500, 513, 2048)])
def test_dense_tile_long_lists_and_depth_ties(rast, oracle_mod, n_distinct, min_len, max_len):
    """Per-tile lists in each sort regime -- beyond the 4096-entry shared-memory sort (chunked
    global/shared bitonic path), the shared-memory bitonic range and the radix range -- with
    exact depth-key ties (duplicated means) that only the source index breaks
    (SPEC.md:270-271): sorted order, ranges, image and gradients vs the oracle."""
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, Scene, grads_as_rows

    rng = np.random.default_rng(11)
    d = np.array([0.2, 0.1, 1.0]) / np.linalg.norm([0.2, 0.1, 1.0])
    base = d * rng.uniform(3.0, 6.0, size=(n_distinct, 1)) + rng.normal(0, 0.02, size=(n_distinct, 3))
    means = np.repeat(base, 2, axis=0).astype(np.float32)  # every depth key appears twice
    n = means.shape[0]
    q = rng.standard_normal((n, 4))
    sh = np.zeros((n, 48), np.float32)
    sh[:, [0, 16, 32]] = rng.normal(0, 0.3, size=(n, 3))
    sc = Scene(means, (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32),
               rng.normal(-3.0, 0.3, size=(n, 3)).astype(np.float32), rng.normal(-1, 1, size=n).astype(np.float32),
               sh, np.zeros(3, np.float32))
    cam = small_fisheye(320, 240)
    ds = to_device(sc)
    img, st = rast.forward(ds, cam, RenderOptions(sh_degree=0), want_stats=True)
    res = oracle_mod.render(sc, cam, sh_degree=0)
    off = res.get("offsets")
    longest = int(np.diff(off).max())
    assert longest >= min_len and (max_len is None or longest <= max_len), longest
    np.testing.assert_array_equal(rast.debug("offsets"), off)
    np.testing.assert_array_equal(rast.debug("sorted_gauss"), res.get("source")[res.get("refs")])
    torch.cuda.synchronize()
    assert np.abs(img.cpu().numpy().astype(np.float64) - res.image).max() <= 1e-3
    dl = rng.standard_normal((cam.height, cam.width, 3)).astype(np.float32)
    g = rast.backward(ds, cam, torch.from_numpy(dl).cuda(), BackwardOptions())
    torch.cuda.synchronize()
    ref, _ = oracle_mod.backward(res, sc.n, dl)
    got = grads_as_rows(g, sc.n)
    for k in ("mean", "rotation", "log_scale", "opacity", "sh_dc"):
        assert rel_l2(got[:, GROUPS[k]], ref[:, GROUPS[k]]) <= 1e-3, k


def test_capacity_growth_and_speculative_launch(rast, oracle_mod):
    """The scatter/sort/blend kernels are launched before the host knows I, against the
    capacity of the previous frames' buffers; a frame whose I exceeds it must be relaunched
    with grown buffers. Small -> large -> small -> large scenes on one context, each checked."""
    import torch
    from paper_2409_04751_b200 import Rasterizer, RenderOptions, synthetic

    r = Rasterizer(0)
    small, deg, cams, _ = synthetic.config(1, n=3000)
    large, _, _, _ = synthetic.config(1, n=40000)
    cam = cams[0]
    for sc in (small, large, small, large, large):
        img, st = r.forward(to_device(sc), cam, RenderOptions(sh_degree=deg), want_stats=True)
        torch.cuda.synchronize()
        res = oracle_mod.render(sc, cam, sh_degree=deg)
        assert st.num_intersections == res.num_intersections
        np.testing.assert_array_equal(r.debug("offsets"), res.get("offsets"))
        np.testing.assert_array_equal(r.debug("sorted_gauss"), res.get("source")[res.get("refs")])
        assert np.abs(img.cpu().numpy().astype(np.float64) - res.image).max() <= 1e-3


@pytest.mark.parametrize("deg", [3, 2, 1, 0])
def test_zero_copy_host_path_equals_device_path(rast, deg):
    """Pinned host scene arrays are read in place over PCIe by K1 / K4b (fgs_render_host,
    fgs_backward_host): K1 stages geometry per CTA and fetches each SH degree's rows
    warp-cooperatively; results equal the device-resident path bit for bit at every degree and
    at scene sizes that end mid-CTA, and the library reports the bytes it moved."""
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, Scene, grads_as_rows, synthetic

    sc, _, cams, dls = synthetic.config(1, n=30000 + 7 * deg)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory().numpy()
    hs = Scene(pin(sc.means), pin(sc.rotations), pin(sc.log_scales), pin(sc.opacity_logits), pin(sc.sh),
               sc.background)
    img_h, radii, st = rast.render_host(hs, cams[0], RenderOptions(sh_degree=deg))
    t = rast.last_transfer()
    assert t["h2d"] < sc.n * 59 * 4 and t["h2d"] >= sc.n * 40  # zero copy: not the whole scene
    g_h = rast.backward_host(hs, cams[0], dls[0], BackwardOptions())
    ds = to_device(sc)
    img_d, _ = rast.forward(ds, cams[0], RenderOptions(sh_degree=deg))
    g_d = rast.backward(ds, cams[0], torch.from_numpy(dls[0]).cuda(), BackwardOptions())
    torch.cuda.synchronize()
    assert img_h.tobytes() == img_d.cpu().numpy().tobytes()
    assert g_h.tobytes() == g_d.cpu().numpy().tobytes()
    # pageable arrays take the copy path and agree too
    img_p, _, _ = rast.render_host(sc.astype(np.float32), cams[0], RenderOptions(sh_degree=deg))
    assert rast.last_transfer()["h2d"] == sc.n * 59 * 4
    assert img_p.tobytes() == img_h.tobytes()


def test_many_streams_and_interleaved_contexts(rast):
    """The frame's scalars reach the host through a mapped block K2 writes (sequence number +
    hash, no copy on a stream): with many application streams (more than the GPU's hardware
    queues), two contexts rendering alternately, and a context moved between streams, every
    frame's image, statistics and gradients equal a lone context's."""
    import torch
    from paper_2409_04751_b200 import BackwardOptions, Rasterizer, RenderOptions, synthetic

    sc, deg, cams, dls = synthetic.config(2, n=80000)
    ds = to_device(sc)
    dl = torch.from_numpy(dls[0]).cuda()
    o = RenderOptions(sh_degree=deg)
    img0, st0 = rast.forward(ds, cams[0], o, want_stats=True)
    g0 = rast.backward(ds, cams[0], dl, BackwardOptions()).clone()
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(24)]
    for s_ in streams:  # keep them busy-ish
        with torch.cuda.stream(s_):
            torch.zeros(1024, device="cuda").add_(1.0)
    a, b = Rasterizer(0), Rasterizer(0)
    for k in range(6):
        for r in (a, b):
            if k % 2:
                r.set_stream(streams[k].cuda_stream)
            img, st = r.forward(ds, cams[0], o, want_stats=True)
            g = r.backward(ds, cams[0], dl, BackwardOptions())
            torch.cuda.synchronize()
            assert img.cpu().numpy().tobytes() == img0.cpu().numpy().tobytes()
            assert st.num_intersections == st0.num_intersections and st.num_splats == st0.num_splats
            assert torch.equal(g, g0)
    # a frame with a different camera in between: its own statistics, then back
    import dataclasses

    moved = dataclasses.replace(cams[0], translation_wc=np.asarray(cams[0].translation_wc, np.float32) + np.float32(0.3))
    img1, st1 = a.forward(ds, moved, o, want_stats=True)
    torch.cuda.synchronize()
    assert st1.num_intersections != st0.num_intersections
    img2, st2 = a.forward(ds, cams[0], o, want_stats=True)
    torch.cuda.synchronize()
    assert st2.num_intersections == st0.num_intersections
    assert img2.cpu().numpy().tobytes() == img0.cpu().numpy().tobytes()


def test_render_host_async_stream_of_frames(rast):
    """fgs_render_host_async: frames queued back to back (two device images alternating, the
    read-back of one overlapping the next frame's scene reads) give, after fgs_wait, the same
    images, radii and statistics as the blocking call, frame by frame; a blocking call after
    asynchronous ones sees them complete."""
    import dataclasses

    import torch
    from paper_2409_04751_b200 import RenderOptions, Scene, synthetic

    sc, deg, cams, _ = synthetic.config(1, n=50000)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory().numpy()
    hs = Scene(pin(sc.means), pin(sc.rotations), pin(sc.log_scales), pin(sc.opacity_logits), pin(sc.sh),
               sc.background)
    o = RenderOptions(sh_degree=deg)
    views = [dataclasses.replace(cams[0], translation_wc=np.asarray(cams[0].translation_wc, np.float32)
                                 + np.float32(0.05 * k)) for k in range(5)]
    ref = [rast.render_host(hs, v, o) for v in views]
    outs = []
    for v in views:
        img = torch.empty((v.height, v.width, 3), dtype=torch.float32).pin_memory().numpy()
        outs.append(rast.render_host_async(hs, v, o, radii=True, image=img))
    rast.wait()
    for (img, radii, st), (ri, rr, rs) in zip(outs, ref):
        assert img.tobytes() == ri.tobytes()
        assert np.array_equal(radii, rr)
        assert st.num_intersections == rs.num_intersections
    # asynchronous frames, then a blocking one without an explicit wait
    img_a = torch.empty_like(torch.from_numpy(ref[0][0])).pin_memory().numpy()
    rast.render_host_async(hs, views[1], o, image=img_a)
    img_b, _, _ = rast.render_host(hs, views[2], o)
    assert img_a.tobytes() == ref[1][0].tobytes() and img_b.tobytes() == ref[2][0].tobytes()


def test_backward_host_async_stream_of_frames(rast):
    """fgs_backward_host_async after fgs_render_host_async, frame after frame (image and gradient
    read-backs on the copy stream, double-buffered on the device): after fgs_wait every frame's
    gradients equal the blocking calls' bit for bit, accumulate mode included."""
    import dataclasses

    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, Scene, synthetic

    sc, deg, cams, dls = synthetic.config(1, n=40000)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory().numpy()
    hs = Scene(pin(sc.means), pin(sc.rotations), pin(sc.log_scales), pin(sc.opacity_logits), pin(sc.sh),
               sc.background)
    o = RenderOptions(sh_degree=deg)
    views = [dataclasses.replace(cams[0], translation_wc=np.asarray(cams[0].translation_wc, np.float32)
                                 + np.float32(0.04 * k)) for k in range(4)]
    dl = pin(dls[0])
    ref = []
    for v in views:
        rast.render_host(hs, v, o)
        ref.append(rast.backward_host(hs, v, dl, BackwardOptions()).copy())
    outs = []
    for v in views:
        img = torch.empty((v.height, v.width, 3), dtype=torch.float32).pin_memory().numpy()
        g = torch.zeros(59 * sc.n, dtype=torch.float32).pin_memory().numpy()
        rast.render_host_async(hs, v, o, image=img)
        outs.append(rast.backward_host_async(hs, v, dl, BackwardOptions(), grads=g))
    rast.wait()
    for g, r in zip(outs, ref):
        assert g.tobytes() == r.tobytes()
    # accumulate: two views summed through the asynchronous calls equal the blocking sum
    acc = torch.zeros(59 * sc.n, dtype=torch.float32).pin_memory().numpy()
    rast.render_host_async(hs, views[0], o, image=torch.empty((views[0].height, views[0].width, 3)).pin_memory().numpy())
    rast.backward_host_async(hs, views[0], dl, BackwardOptions(), grads=acc)
    rast.wait()
    rast.render_host_async(hs, views[1], o, image=torch.empty((views[1].height, views[1].width, 3)).pin_memory().numpy())
    rast.backward_host_async(hs, views[1], dl, BackwardOptions(), grads=acc, accumulate=True)
    rast.wait()
    acc_ref = ref[0].copy()
    rast.render_host(hs, views[1], o)
    rast.backward_host(hs, views[1], dl, BackwardOptions(), grads=acc_ref, accumulate=True)
    assert acc.tobytes() == acc_ref.tobytes()


@pytest.mark.parametrize("scatter", ["local", "slots", "rows"])
def test_huge_splats_every_binning_path(rast, oracle_mod, scatter):
    """Splats that each cover most of the tile grid: every binning CTA scatters more than one
    8192-intersection pass (bin_local_kernel's multi-pass scatter, the global slot order's
    sub-ranges, the tile-row lists' windows), against the oracle's ranges, order and image."""
    import torch
    from paper_2409_04751_b200 import RenderOptions, Scene, _lib

    rng = np.random.default_rng(21)
    n = 2000
    d = rng.standard_normal((n, 3)) * np.array([0.15, 0.15, 0.0]) + np.array([0.0, 0.0, 1.0])
    means = (d / np.linalg.norm(d, axis=1, keepdims=True) * rng.uniform(4.0, 8.0, size=(n, 1))).astype(np.float32)
    q = rng.standard_normal((n, 4))
    sh = np.zeros((n, 48), np.float32)
    sh[:, [0, 16, 32]] = rng.normal(0, 0.3, size=(n, 3))
    sc = Scene(means, (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32),
               rng.normal(0.6, 0.2, size=(n, 3)).astype(np.float32), rng.normal(-4.0, 0.5, size=n).astype(np.float32),
               sh, np.zeros(3, np.float32))
    cam = small_fisheye(640, 480)
    flags = {"local": _lib.FGS_FLAG_SLOT_SCATTER, "slots": _lib.FGS_FLAG_SLOT_SCATTER | _lib.FGS_FLAG_GLOBAL_SLOTS,
             "rows": _lib.FGS_FLAG_ROW_SCATTER}[scatter]
    rast.set_flags(flags)
    try:
        img, st = rast.forward(to_device(sc), cam, RenderOptions(sh_degree=0), want_stats=True)
        torch.cuda.synchronize()
        vv = rast.debug("variants")
        assert vv[4] == (scatter == "rows") and vv[5] == (scatter == "local")
        res = oracle_mod.render(sc, cam, sh_degree=0)
        assert st.num_intersections == res.num_intersections
        assert res.num_intersections > 148 * 8192  # > one scatter pass per binning CTA
        np.testing.assert_array_equal(rast.debug("offsets"), res.get("offsets"))
        np.testing.assert_array_equal(rast.debug("sorted_gauss"), res.get("source")[res.get("refs")])
        assert np.abs(img.cpu().numpy().astype(np.float64) - res.image).max() <= 1e-3
    finally:
        rast.set_flags(0)
