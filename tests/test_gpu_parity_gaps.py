"""GPU parity cases that target specific branches and hot-path state (round-2 additions).

* fisheye Taylor-series branch (l_z^2 < 1e-6 z^2, /root/reference/proj/include/omnisplat/
  cameras.hpp:104-117) and the exactly-on-axis point (l_z = 0, where the general path would divide
  by zero), pinned in the reference at tests/test_cameras.cpp:137-143 and :287-318;
* config 1 at its BASELINE size (200k Gaussians), forward + backward;
* the pre-sort key list taken from the hot path's own state (K2's compaction + scatter output),
  not from a debug reconstruction kernel, at config 2 full scale;
* the blend work counters E_eval / E_contrib (which feed every roofline) at config 2;
* the multi-view gradient sum of config 4: GPU accumulation over views
  against the sum of per-view oracle gradients, and the 8-view accumulation against a float64 sum
  of 8 single-view GPU backwards.
"""
import numpy as np
import pytest

from tests._helpers import GROUPS, rel_l2, to_device
from tests.test_gpu_parity import (check_grads, check_image, check_keys, check_preprocess, run_gpu, run_oracle)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rast():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2409_04751_b200 import Rasterizer

    return Rasterizer(0)


def axis_scene(seed=11):
    """Gaussians on and near the optical axis of an identity-pose fisheye: exactly on the axis in
    front (l_z = 0: series branch), exactly on the axis behind (invisible), and a log-uniform band
    l_z / z in [1e-4, 2e-3] that straddles the series/general switch at 1e-3, including points
    placed on the switch itself."""
    from paper_2409_04751_b200 import Scene

    rng = np.random.default_rng(seed)
    parts = []
    z_on = rng.uniform(0.8, 8.0, 48)
    parts.append(np.stack([np.zeros(48), np.zeros(48), z_on], 1))
    z_back = rng.uniform(0.8, 8.0, 8)
    parts.append(np.stack([np.zeros(8), np.zeros(8), -z_back], 1))
    nb = 320
    z = rng.uniform(0.8, 8.0, nb)
    rho = 10 ** rng.uniform(-4.0, np.log10(2e-3), nb)
    phi = rng.uniform(0, 2 * np.pi, nb)
    parts.append(np.stack([rho * z * np.cos(phi), rho * z * np.sin(phi), z], 1))
    # on the switch: x = 1e-3 z (and its float neighbours), y = 0 / x = 0
    zs = rng.uniform(1.0, 6.0, 16).astype(np.float32)
    xs = (np.float32(1e-3) * zs).astype(np.float32)
    edge = [np.stack([np.nextafter(xs, np.float32(d)) if d else xs, np.zeros(16, np.float32), zs], 1)
            for d in (0, -1, 1)]
    edge.append(np.stack([np.zeros(16, np.float32), xs, zs], 1))
    parts += edge
    means = np.concatenate(parts).astype(np.float32)
    n = len(means)
    rot = rng.standard_normal((n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    ls = rng.normal(-3.0, 0.4, (n, 3))
    op = rng.normal(0.5, 1.0, n)
    sh = np.zeros((n, 3, 16))
    sh[:, :, 0] = rng.normal(0.0, 0.3, (n, 3))
    sh[:, :, 1:] = rng.normal(0.0, 0.05, (n, 3, 15))
    f = lambda a: np.ascontiguousarray(a, np.float32)
    return Scene(f(means), f(rot), f(ls), f(op), f(sh.reshape(n, 48)), np.zeros(3, np.float32))


@pytest.mark.parametrize("fov_deg", [90.0, 100.0])
def test_on_axis_and_series_band_parity(rast, oracle_mod, fov_deg):
    from paper_2409_04751_b200 import Camera

    scene = axis_scene()
    w, h = 320, 256
    fov = np.radians(fov_deg)
    f = 0.5 * np.hypot(w, h) / fov
    cam = Camera.fisheye(w, h, f, f, w / 2, h / 2, fov).as_float32()
    m = scene.means.astype(np.float32)
    lz2 = m[:, 0] * m[:, 0] + m[:, 1] * m[:, 1]
    z2 = m[:, 2] * m[:, 2]
    series = (m[:, 2] > 0) & (lz2 < np.float32(1e-6) * z2)
    assert series.sum() >= 100 and (~series & (m[:, 2] > 0)).sum() >= 100
    assert ((lz2 == 0) & (m[:, 2] > 0)).sum() == 48
    dl = np.random.default_rng(3).standard_normal((h, w, 3)).astype(np.float32)
    g = run_gpu(rast, scene, cam, 3, dl)
    o = run_oracle(oracle_mod, scene, cam, 3, dl)
    state = o["res"].get("state")
    assert (state[:48] == 1).all(), "on-axis Gaussians in front must be kept"
    assert (state[48:56] == 0).all(), "on-axis Gaussians behind the camera are invisible"
    check_preprocess(g, o, scene)
    check_keys(rast, o)
    check_image(g, o)
    check_grads(g, o)
    # the on-axis rows themselves: every gradient finite and non-trivial where they contribute
    assert np.isfinite(g["grads"][:48]).all()
    assert np.abs(g["grads"][:48, 0:3]).sum() > 0


def test_cfg1_full_scale_fwd_bwd_parity(rast, oracle_mod):
    """Config 1 at its BASELINE size: 200,000 Gaussians, SH3, 1752x1168, forward + backward."""
    from paper_2409_04751_b200 import synthetic

    scene, deg, cams, dls = synthetic.config(1)
    assert scene.n == 200_000
    g = run_gpu(rast, scene, cams[0], deg, dls[0])
    o = run_oracle(oracle_mod, scene, cams[0], deg, dls[0])
    check_preprocess(g, o, scene)
    check_keys(rast, o)
    check_image(g, o)
    check_grads(g, o)


@pytest.mark.parametrize("scatter", ["slots", "rows", "local"])
def test_cfg2_hot_path_key_list_and_counters(rast, oracle_mod, scatter):
    """Config 2 full scale (1M clustered Gaussians), with either scatter work order (tile-row
    lists or source-order slots). The pre-sort key list comes from the hot path's own state: K2's compaction (the tile-touching Gaussians in source order with their
    first emission slots) and K1's tile rectangles give the reference's emission order
    (splatting.hpp:216-221), and the 64-bit keys K2's scatter wrote into every tile's range are, per
    tile, exactly the reference's (depth key, source) keys of that tile. Then E_eval / E_contrib
    (the roofline counters) against the oracle's instrumented render."""
    from paper_2409_04751_b200 import RenderOptions, _lib, synthetic

    scene, deg, cams, _ = synthetic.config(2)
    cam = cams[0]
    o = oracle_mod.render(scene, cam, sh_degree=deg, mode=oracle_mod.MODE_PARITY)
    src = o.get("source")
    ref_tile = o.get("key_tile").astype(np.int64)
    ref_depth = o.get("key_depth").astype(np.uint64)
    ref_gauss = src[o.get("key_splat")].astype(np.uint64)
    I = len(ref_tile)
    assert I > 500_000

    ds = to_device(scene)
    force = {"rows": _lib.FGS_FLAG_ROW_SCATTER, "local": _lib.FGS_FLAG_SLOT_SCATTER,
             "slots": _lib.FGS_FLAG_SLOT_SCATTER | _lib.FGS_FLAG_GLOBAL_SLOTS}[scatter]
    rast.set_flags(_lib.FGS_FLAG_COUNTERS | force)
    try:
        _, st = rast.forward(ds, cam, RenderOptions(sh_degree=deg), want_stats=True)
        ev, ec = rast.debug("counters", np.uint64)[:2]
        vv = rast.debug("variants")
        assert vv[4] == (1 if scatter == "rows" else 0) and vv[5] == (1 if scatter == "local" else 0)
    finally:
        rast.set_flags(0)
    assert st.num_intersections == I
    ost = o.stats()
    # The skip / clamp decisions are exact (guard band around 1/255 and 0.99), but the
    # transmittance stop (T' < 1e-4, splatting.hpp:291-292) compares a product of fp32 (1 - alpha)
    # factors whose alphas come from the fast exp (<= 2 ulp): a pixel whose T' lands within ~1e-5
    # relative of 1e-4 may stop one entry earlier or later (at config 2: 9 of 167M evaluations).
    # The counters feed the roofline's work figure, so they are checked to 1e-6 relative.
    assert abs(int(ev) - int(ost["e_eval"])) <= 1e-6 * ost["e_eval"], (int(ev), ost["e_eval"])
    assert abs(int(ec) - int(ost["e_contrib"])) <= 1e-6 * ost["e_contrib"], (int(ec), ost["e_contrib"])

    # emission order from the compaction state
    cval = rast.debug("compact_gauss").astype(np.int64)
    coff = rast.debug("compact_offsets").astype(np.int64)
    rect = rast.debug("rect", np.uint16).reshape(-1, 4).astype(np.int64)[cval]
    wx = rect[:, 1] - rect[:, 0] + 1
    cnt = wx * (rect[:, 3] - rect[:, 2] + 1)
    np.testing.assert_array_equal(coff, np.concatenate([[0], np.cumsum(cnt)[:-1]]))
    assert int(cnt.sum()) == I
    owner = np.repeat(np.arange(len(cval)), cnt)
    j = np.arange(I) - coff[owner]
    tiles_x = cam.tiles_x
    got_tile = (rect[owner, 2] + j // wx[owner]) * tiles_x + rect[owner, 0] + j % wx[owner]
    np.testing.assert_array_equal(got_tile, ref_tile)
    np.testing.assert_array_equal(cval[owner].astype(np.uint64), ref_gauss)

    # the scatter's output, tile by tile, as multisets of 64-bit keys
    keys = rast.debug("keys", np.uint64)
    off = rast.debug("offsets").astype(np.int64)
    np.testing.assert_array_equal(off, o.get("offsets"))
    k_tile = np.repeat(np.arange(len(off) - 1), np.diff(off))
    got = keys[np.lexsort((keys, k_tile))]
    ref_keys = (ref_depth << np.uint64(32)) | ref_gauss
    ref = ref_keys[np.lexsort((ref_keys, ref_tile))]
    np.testing.assert_array_equal(got, ref)
    # and the depth half of each key is K1's key for that Gaussian
    dk = rast.debug("depth_key")
    np.testing.assert_array_equal((keys >> np.uint64(32)).astype(np.uint32), dk[(keys & np.uint64(0xFFFFFFFF)).astype(np.int64)])


def test_cfg4_multiview_accumulated_gradients(rast, oracle_mod):
    """Config 4 (3M Gaussians, 8 views per GPU): the accumulating backward (accumulate=1 into one
    59*N buffer, what one rank does before the all-reduce) equals the sum of per-view oracle
    gradients on 2 views (rel-L2 <= 1e-3 per group), and the 8-view accumulation equals the float64
    sum of 8 separate single-view GPU backwards to fp32 summation order (rel-L2 <= 1e-6)."""
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, grads_as_rows, synthetic

    scene, deg, cams, dls = synthetic.config(4)
    assert len(cams) == 8
    n = scene.n
    ds = to_device(scene)
    ro = RenderOptions(sh_degree=deg)
    acc = torch.zeros(59 * n, dtype=torch.float32, device="cuda")
    single = torch.zeros(59 * n, dtype=torch.float32, device="cuda")
    total = torch.zeros(59 * n, dtype=torch.float64, device="cuda")
    acc2 = None
    for v in range(8):
        dl = torch.from_numpy(dls[v]).cuda()
        rast.forward(ds, cams[v], ro)
        rast.backward(ds, cams[v], dl, BackwardOptions(), grads=acc, accumulate=v > 0)
        rast.backward(ds, cams[v], dl, BackwardOptions(), grads=single, accumulate=False)
        total += single.double()
        if v == 1:
            acc2 = grads_as_rows(acc, n)
    torch.cuda.synchronize()
    got8 = acc.double()
    assert rel_l2(got8.cpu().numpy(), total.cpu().numpy()) <= 1e-6
    del got8, total, single

    ref = None
    for v in range(2):
        res = oracle_mod.render(scene, cams[v], sh_degree=deg, mode=oracle_mod.MODE_PARITY)
        gv, _ = oracle_mod.backward(res, n, dls[v], mode=oracle_mod.MODE_PARITY)
        res.close()
        ref = gv.astype(np.float64) if ref is None else ref + gv
    for k in ("mean", "rotation", "log_scale", "opacity", "sh_dc", "sh_rest"):
        e = rel_l2(acc2[:, GROUPS[k]], ref[:, GROUPS[k]])
        assert e <= 1e-3, (k, e)


def test_odd_n_flat_buffer_alignment(rast, oracle_mod):
    """Scene arrays that are field blocks of one flat 59*N buffer with N % 4 != 0 (rotations at
    byte 12N, SH at byte 44N: not 16-byte aligned) -- the layout Trainer.params uses. The
    vectorised loads fall back to scalar loads; results equal the aligned case."""
    import torch
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions, Scene, grads_as_rows, synthetic

    scene, deg, cams, dls = synthetic.config(1, n=1001)
    n = scene.n
    flat = torch.cat([torch.from_numpy(np.ascontiguousarray(a, np.float32)).reshape(-1)
                      for a in (scene.means, scene.rotations, scene.log_scales, scene.opacity_logits, scene.sh)]).cuda()
    parts, off = [], 0
    for wdt in (3, 4, 3, 1, 48):
        parts.append(flat[off:off + wdt * n].view(n, wdt) if wdt > 1 else flat[off:off + n])
        off += wdt * n
    ds_flat = Scene(*parts, scene.background)
    assert parts[1].data_ptr() % 16 != 0 and parts[4].data_ptr() % 16 != 0
    ro = RenderOptions(sh_degree=deg)
    img_a = rast.forward(ds_flat, cams[0], ro)[0].clone()
    dl = torch.from_numpy(dls[0]).cuda()
    ga = grads_as_rows(rast.backward(ds_flat, cams[0], dl, BackwardOptions()), n)
    ds = to_device(scene)
    img_b = rast.forward(ds, cams[0], ro)[0].clone()
    gb = grads_as_rows(rast.backward(ds, cams[0], dl, BackwardOptions()), n)
    torch.cuda.synchronize()
    assert torch.equal(img_a, img_b)
    np.testing.assert_array_equal(ga, gb)


def test_fast_correctly_rounded_math():
    """csrc/fgs_crmath.cuh (K1 / K4b): the fast exp equals cr_expf on every one of the 2^32 fp32
    inputs; the fast atan2 equals cr_atan2f on 2^28 random bit-pattern pairs and 2^28 pairs of
    the camera domain; the slow path is rare (the exp's bound: < 1e-6 of finite in-range inputs)."""
    from paper_2409_04751_b200 import Rasterizer

    r = Rasterizer(0)
    e = r.selftest_crmath(0, 0, 1 << 32)
    assert e["checked"] == 1 << 32 and e["mismatches"] == 0, e
    # slow path: |x| > 87, NaN, inf (every pattern above 87.0 = 0x42AE0000 in magnitude) plus the
    # near-midpoint band of the in-range inputs
    in_range = 2 * (0x42AE0000 + 1)
    assert 0 <= e["slow"] - ((1 << 32) - in_range) < 1e-5 * in_range, e
    for which, seed in ((1, 1), (2, 2)):
        a = r.selftest_crmath(which, 0, 1 << 28, seed)
        assert a["checked"] == 1 << 28 and a["mismatches"] == 0, (which, a)
    cam = r.selftest_crmath(2, 0, 1 << 28, 3)
    assert cam["slow"] < 5e-4 * cam["checked"], cam  # (1/1088 of the pairs have y = 0 exactly)
