"""Backward pins of the CPU oracle, ported from the reference's gradient tests
(/root/reference/proj/tests/test_gradients.cpp, test_oracle.cpp) and its gradcheck machinery
(inc/oracle.hpp:338-566), plus the build's extension: FD pins for the 45 higher-band SH
gradients, which the reference does not implement (SURVEY.md §0 gap 1, "parity unpinned" in the
reference sense; pinned here by finite differences of the double brute-force renderer).
"""
import math

import numpy as np
import pytest

import oracle
from paper_2409_04751_b200 import Camera, Scene


def angle_axis(angle, axis):
    a = np.asarray(axis, float)
    a /= np.linalg.norm(a)
    x, y, z = a
    c, s, t = math.cos(angle), math.sin(angle), 1 - math.cos(angle)
    return np.array([[t * x * x + c, t * x * y - s * z, t * x * z + s * y],
                     [t * x * y + s * z, t * y * y + c, t * y * z - s * x],
                     [t * x * z - s * y, t * y * z + s * x, t * z * z + c]])


def gradcheck_camera(model):
    if model == "pinhole":
        cam = Camera.pinhole(32, 32, 24.0, 24.0, 16.0, 16.0)
    elif model == "fisheye":
        cam = Camera.fisheye(32, 32, 9.5, 9.5, 16.0, 16.0, math.pi / 2)
    else:
        cam = Camera.panorama(64, 32)
    cam.rotation_wc = angle_axis(0.3, [0.2, 1.0, 0.5])
    cam.translation_wc = np.array([0.1, -0.2, 0.3])
    return cam


def make_gradcheck_scene(model, seed, n, wide_angle=True, sh_rest=0.0):
    """inc/oracle.hpp:425-566: candidates are rejected until every blend decision, radius and
    depth order sits a safe margin away from its threshold."""
    rng = np.random.default_rng(seed ^ 0x9E3779B97F4A7C15)
    cam = gradcheck_camera(model)
    W, b = cam.rotation_wc, cam.translation_wc
    for _ in range(400):
        means, ls, rots, ops, shs = [], [], [], [], []
        for i in range(n):
            if model == "pinhole":
                z = rng.uniform(3.0, 5.0)
                pc = np.array([rng.uniform(-0.45, 0.45) * z, rng.uniform(-0.45, 0.45) * z, z])
                base = rng.uniform(0.20, 0.42)
            elif model == "fisheye":
                th = rng.uniform(0.10, 1.45)
                if wide_angle and i == 0:
                    th = rng.uniform(math.radians(80.0), math.radians(85.0))
                ph, d = rng.uniform(0, 2 * math.pi), rng.uniform(2.5, 4.5)
                pc = d * np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
                base = rng.uniform(0.50, 0.90)
            else:
                lon, lat, d = rng.uniform(-2.4, 2.4), rng.uniform(-0.9, 0.9), rng.uniform(2.5, 4.5)
                pc = d * np.array([math.cos(lat) * math.sin(lon), math.sin(lat), math.cos(lat) * math.cos(lon)])
                base = rng.uniform(0.45, 0.85)
            means.append(W.T @ (pc - b))
            while True:
                an = rng.uniform(0.75, 1.35, 3)
                if an.max() / an.min() >= 1.15:
                    break
            ls.append(np.log(base * an))
            while True:
                q = rng.uniform(-1, 1, 4)
                if np.linalg.norm(q) >= 0.1:
                    break
            rots.append(q / np.linalg.norm(q) * rng.uniform(0.7, 1.3))
            p = rng.uniform(0.10, 0.28)
            ops.append(math.log(p / (1 - p)))
            sh = np.zeros(48)
            sh[[0, 16, 32]] = rng.uniform(-1.0, 1.0, 3)
            if sh_rest:
                sh += rng.uniform(-sh_rest, sh_rest, 48) * (np.arange(48) % 16 != 0)
            shs.append(sh)
        scene = Scene(np.array(means), np.array(rots), np.array(ls), np.array(ops), np.array(shs),
                      np.array([0.15, 0.20, 0.25]))
        if _threshold_safe(scene, cam, n):
            return scene, cam
    raise RuntimeError("make_gradcheck_scene: no threshold-safe configuration found")


def _threshold_safe(scene, cam, n):
    res = oracle.render(scene, cam, sh_degree=0, dtype=np.float64, threads=1)
    if res.num_splats != n:
        return False
    m = res.get("mean_px").reshape(-1, 2)
    con = res.get("conic").reshape(-1, 3)
    rad = res.get("radius")
    dep = res.get("depth")
    al = res.get("alpha")
    for i in range(n):  # radius away from the next integer
        a, bb, c = con[i]
        det = a * c - bb * bb
        sa, sc, sb = c / det, a / det, -bb / det
        mid = 0.5 * (sa + sc)
        lmax = mid + math.sqrt(max(mid * mid - (sa * sc - sb * sb), 0.0))
        rexact = 3.0 * math.sqrt(lmax)
        frac = rexact - math.floor(rexact)
        if frac < 0.03 or frac > 0.97:
            return False
    for i in range(n):  # depth separation of overlapping splats
        for j in range(i + 1, n):
            ov = abs(m[i, 0] - m[j, 0]) <= rad[i] + rad[j] and abs(m[i, 1] - m[j, 1]) <= rad[i] + rad[j]
            if ov and abs(dep[i] - dep[j]) < 5e-4:
                return False
    off, refs = res.get("offsets"), res.get("refs")
    for t in range(len(off) - 1):
        lo, hi = off[t], off[t + 1]
        if lo == hi:
            continue
        tx, ty = t % res.tiles_x, t // res.tiles_x
        for py in range(ty * 16, min(cam.height, ty * 16 + 16)):
            for px in range(tx * 16, min(cam.width, tx * 16 + 16)):
                trans = 1.0
                for k in range(lo, hi):
                    s = refs[k]
                    dx, dy = px + 0.5 - m[s, 0], py + 0.5 - m[s, 1]
                    power = -0.5 * (con[s, 0] * dx * dx + con[s, 2] * dy * dy) - con[s, 1] * dx * dy
                    if power > 0:
                        continue
                    ar = al[s] * math.exp(power)
                    if abs(ar - 1 / 255) < 1e-5 or ar >= 0.9 * 0.99:
                        return False
                    if ar < 1 / 255:
                        continue
                    nt = trans * (1 - ar)
                    if abs(nt - 1e-4) < 1e-6:
                        return False
                    if nt < 1e-4:
                        break
                    trans = nt
                if trans < 5e-4:
                    return False
    return True


def sum_squares_grad(img):
    return 2.0 * img


def gradcheck(scene, cam, step=1e-4, tol=1e-3, jacobian_grad_scale=None, sh_degree=0, params="dc", view_dir=False):
    """inc/oracle.hpp:338-418: analytic backward of L = sum(pixel^2) vs central differences of the
    brute-force renderer's loss. params='dc' checks the reference's 14 per-Gaussian parameters;
    'rest' the 45 higher-band SH coefficients (build extension)."""
    res = oracle.render(scene, cam, sh_degree=sh_degree, dtype=np.float64, threads=1)
    g, _ = oracle.backward(res, scene.n, sum_squares_grad(res.image), full_sh=True,
                           jacobian_grad_scale=jacobian_grad_scale, sh_view_dir_grad=view_dir)
    if params == "dc":
        cols = list(range(11)) + [11, 27, 43]
        names = {"mean": range(0, 3), "rotation": range(3, 7), "log_scale": range(7, 10), "opacity": [10],
                 "sh_dc": [11, 27, 43]}
    else:
        cols = [11 + c * 16 + j for c in range(3) for j in range(1, 16)]
        names = {"sh_rest": cols}
    fd = np.zeros_like(g)

    def loss(s):
        img, _ = oracle.bruteforce_render(s, cam, sh_degree=sh_degree)
        return float((img ** 2).sum())

    fields = [("means", 3), ("rotations", 4), ("log_scales", 3), ("opacity_logits", 1), ("sh", 48)]
    for gi in range(scene.n):
        for col in cols:
            acc, fi = 0, 0
            while col >= acc + fields[fi][1]:
                acc += fields[fi][1]
                fi += 1
            name, k = fields[fi][0], col - acc
            vals = []
            for d in (step, -step):
                s = Scene(*(np.array(getattr(scene, f), float) for f in
                            ("means", "rotations", "log_scales", "opacity_logits", "sh")), scene.background)
                arr = getattr(s, name)
                if arr.ndim == 1:
                    arr[gi] += d
                else:
                    arr[gi, k] += d
                vals.append(loss(s))
            fd[gi, col] = (vals[0] - vals[1]) / (2 * step)
    report = {}
    for grp, cs in names.items():
        worst = 0.0
        for gi in range(scene.n):
            for c in cs:
                a, b = g[gi, c], fd[gi, c]
                worst = max(worst, abs(a - b) / max(abs(a), abs(b), 1e-8))
        report[grp] = worst
    return report, all(v < tol for v in report.values())


# ------------------------------------------------------------------ tests/test_gradients.cpp

def test_zero_image_gradient_gives_zero():  # test_gradients.cpp:46-57, :257-285
    scene, cam = make_gradcheck_scene("fisheye", 11, 6)
    culled_pos = cam.rotation_wc.T @ (np.array([0, 0, -5.0]) - cam.translation_wc)
    scene = Scene(np.vstack([scene.means, culled_pos]), np.vstack([scene.rotations, [1, 0, 0, 0]]),
                  np.vstack([scene.log_scales, [0, 0, 0]]), np.append(scene.opacity_logits, 0.0),
                  np.vstack([scene.sh, np.zeros(48)]), scene.background)
    res = oracle.render(scene, cam, sh_degree=0, dtype=np.float64)
    assert res.stats()["num_culled"] == 1
    g0, sg = oracle.backward(res, scene.n, np.zeros((32, 32, 3)), want_splat_grads=True)
    assert not g0.any() and not sg.any()
    g, _ = oracle.backward(res, scene.n, sum_squares_grad(res.image))
    assert not g[-1].any() and np.isfinite(g).all()


def test_color_gradient_is_blended_weight():  # test_gradients.cpp:59-93
    r = oracle.splats_render([[8.5, 8.5]], [[0.5, 0.0, 0.5]], [1.0], [4], [[0.8, 0.3, 0.1]], [0.9], 16, 16)
    dl = np.zeros((16, 16, 3))
    dl[:, :, 0] = 1.0
    sg = oracle.splats_backward(r, dl)
    wsum = (1.0 - r.get("final_T")).sum()
    assert sg[0, 5] == pytest.approx(wsum, rel=1e-12)
    assert sg[0, 6] == 0.0 and sg[0, 7] == 0.0


def test_rasterize_backward_matches_fd():  # test_gradients.cpp:95-138
    scene, cam = make_gradcheck_scene("pinhole", 77, 8)
    res = oracle.render(scene, cam, sh_degree=3, dtype=np.float64)
    sg = oracle.splats_backward(res, sum_squares_grad(res.image))
    base = {k: res.get(k) for k in ("mean_px", "conic", "depth", "radius", "color", "alpha")}
    base["mean_px"] = base["mean_px"].reshape(-1, 2)
    base["conic"] = base["conic"].reshape(-1, 3)
    base["color"] = base["color"].reshape(-1, 3)
    h = 1e-5

    def loss(sp):
        r = oracle.splats_render(sp["mean_px"], sp["conic"], sp["depth"], sp["radius"], sp["color"], sp["alpha"],
                                 cam.width, cam.height, scene.background)
        return float((r.image ** 2).sum())

    worst = 0.0
    fields = [("mean_px", 2), ("conic", 3), ("color", 3), ("alpha", 1)]
    for i in range(res.num_splats):
        col = 0
        for name, k in fields:
            for c in range(k):
                vals = []
                for d in (h, -h):
                    sp = {kk: np.array(v, copy=True) for kk, v in base.items()}
                    if sp[name].ndim == 1:
                        sp[name][i] += d
                    else:
                        sp[name][i, c] += d
                    vals.append(loss(sp))
                fd = (vals[0] - vals[1]) / (2 * h)
                a = sg[i, col]
                worst = max(worst, abs(a - fd) - (1e-6 * max(abs(a), abs(fd)) + 1e-7))
                col += 1
    assert worst <= 0.0


def test_backward_rejects_mismatched_scene():  # test_gradients.cpp:287-299
    scene, cam = make_gradcheck_scene("pinhole", 3, 4)
    res = oracle.render(scene, cam, dtype=np.float64)
    with pytest.raises(oracle.OracleError, match="different scene"):
        oracle.backward(res, scene.n - 1, np.zeros((32, 32, 3)))


@pytest.mark.parametrize("model", ["pinhole", "fisheye", "panorama"])
def test_end_to_end_gradcheck(model):  # test_gradients.cpp:301-310
    scene, cam = make_gradcheck_scene(model, 42, 6)
    report, ok = gradcheck(scene, cam)
    assert ok, report


def test_wide_angle_fisheye_gradcheck_and_mutation():  # test_oracle.cpp:122-149
    scene, cam = make_gradcheck_scene("fisheye", 57, 10)
    pc = (cam.rotation_wc @ scene.means.T).T + cam.translation_wc
    assert np.arctan2(np.hypot(pc[:, 0], pc[:, 1]), pc[:, 2]).max() > math.radians(80.0)
    report, ok = gradcheck(scene, cam)
    assert ok, report
    for k in range(3):
        s = [1.0, 1.0, 1.0]
        s[k] = 1.1
        report, ok = gradcheck(scene, cam, jacobian_grad_scale=s)
        assert not ok and report["mean"] >= 1e-3, (k, report)


def test_gradcheck_simple_pinhole_at_1e6():  # test_oracle.cpp:107-114
    scene, cam = make_gradcheck_scene("pinhole", 21, 1)
    report, ok = gradcheck(scene, cam, tol=1e-6)
    assert ok, report


def test_mean_gradient_is_sum_of_paths():  # test_gradients.cpp:312-344
    """With the covariance path's dJ/dmu scaled to zero the mean gradient is the direct path;
    the full gradient minus it is the covariance path, and both are non-zero."""
    scene, cam = make_gradcheck_scene("fisheye", 31, 6)
    res = oracle.render(scene, cam, sh_degree=0, dtype=np.float64)
    dl = sum_squares_grad(res.image)
    full, _ = oracle.backward(res, scene.n, dl)
    direct_plus_sigma, _ = oracle.backward(res, scene.n, dl, jacobian_grad_scale=[0, 0, 0])
    cov_path = full[:, 0:3] - direct_plus_sigma[:, 0:3]
    assert np.abs(cov_path).sum() > 0 and np.abs(direct_plus_sigma[:, 0:3]).sum() > 0
    doubled, _ = oracle.backward(res, scene.n, dl, jacobian_grad_scale=[2, 2, 2])
    np.testing.assert_allclose(doubled[:, 0:3] - full[:, 0:3], cov_path, rtol=1e-9, atol=1e-12)


def test_backward_deterministic_across_threads():  # test_gradients.cpp:426-446
    scene, cam = make_gradcheck_scene("fisheye", 63, 8)
    for dt in (np.float64, np.float32):
        res = oracle.render(scene, cam, sh_degree=0, dtype=dt)
        dl = sum_squares_grad(res.image)
        a, _ = oracle.backward(res, scene.n, dl, threads=1)
        b, _ = oracle.backward(res, scene.n, dl, threads=1)
        c, _ = oracle.backward(res, scene.n, dl, threads=5)
        assert a.tobytes() == b.tobytes() == c.tobytes()


# ------------------------------------------------------------ build extension: SH rest bands

def test_sh_rest_band_gradients_fd():
    """The 45 higher-band SH gradients (not in the reference) against FD of the double
    brute-force renderer at sh_degree 3."""
    scene, cam = make_gradcheck_scene("fisheye", 42, 4, sh_rest=0.3)
    report, ok = gradcheck(scene, cam, sh_degree=3, params="rest")
    assert ok, report


def test_sh_view_direction_mean_gradient():
    """SURVEY.md §0 gap 2: the reference drops colour -> view direction -> mean. At SH degree 3
    its mean gradient therefore misses FD (kept as the default, for reference parity); the
    opt-in sh_view_dir_grad path passes the full 14-parameter gradcheck."""
    scene, cam = make_gradcheck_scene("fisheye", 42, 4, sh_rest=0.3)
    report, ok = gradcheck(scene, cam, sh_degree=3, params="dc")
    assert not ok and report["mean"] > 1e-3 and all(v < 1e-3 for k, v in report.items() if k != "mean")
    report, ok = gradcheck(scene, cam, sh_degree=3, params="dc", view_dir=True)
    assert ok, report
