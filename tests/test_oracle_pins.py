"""Pins the CPU oracle (oracle/fgs_oracle.cpp) against the reference's own known-answer and
property tests for this path, ported from /root/reference/proj/tests (cited per test).

The reference's tests draw from std::mt19937_64 streams; the ported property tests draw the
same distributions from numpy instead (the checked properties do not depend on the stream).
Hand-derived goldens are reproduced exactly.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2409_04751_b200 import Camera, Scene
from paper_2409_04751_b200.types import CAMERA_FISHEYE, CAMERA_PANORAMA, CAMERA_PINHOLE

RNG = np.random.default_rng(7)


@pytest.fixture(autouse=True)
def _reseed():
    # each test draws from its own fixed stream (the reference seeds one stream per file)
    global RNG
    RNG = np.random.default_rng(7)


def rel_err(a, b):  # inc/oracle.hpp:39-41
    return abs(a - b) / max(abs(a), abs(b), 1e-8)


def one_gaussian(mean, rot=(1, 0, 0, 0), log_scale=(0, 0, 0), logit=0.0, sh=None):
    shv = np.zeros((1, 48)) if sh is None else np.asarray(sh, np.float64).reshape(1, 48)
    return Scene(np.array([mean], float), np.array([rot], float), np.array([log_scale], float), np.array([logit]),
                 shv, np.zeros(3))


def test_cameras():
    """Camera factories exist for all three models (the oracle keeps pinhole/panorama for the
    ported tests; the GPU path is fisheye-only)."""
    assert Camera.pinhole(4, 4, 1, 1, 2, 2).model == CAMERA_PINHOLE
    assert Camera.panorama(4, 4).model == CAMERA_PANORAMA
    assert Camera.fisheye(4, 4, 1, 1, 2, 2).model == CAMERA_FISHEYE


# ---------------------------------------------------------------- tests/test_cameras.cpp

def test_fisheye_projection_fixed_values():  # test_cameras.cpp:89-103
    cam = Camera.fisheye(400, 300, 100.0, 100.0, 200.0, 150.0)
    v, px, _ = oracle.project(cam, [0, 0, 1])
    assert v and px[0] == pytest.approx(200.0, rel=1e-12) and px[1] == pytest.approx(150.0, rel=1e-12)
    cam.cx = 0.0
    _, px, _ = oracle.project(cam, [1, 0, 1])
    assert px[0] == pytest.approx(100.0 * math.pi / 4, rel=1e-12)
    _, px, _ = oracle.project(cam, [1, 0, 0])
    assert px[0] == pytest.approx(100.0 * math.pi / 2, rel=1e-12)


def test_fisheye_culling_margin():  # test_cameras.cpp:125-135
    cam = Camera.fisheye(640, 480, 190.0, 185.0, 320.0, 240.0, math.pi / 2)
    at = lambda deg: oracle.project(cam, [math.sin(math.radians(deg)), 0, math.cos(math.radians(deg))])[0]
    assert at(85) and at(99) and not at(101) and not at(120)


def test_on_axis_fisheye_jacobian_is_pinhole():  # test_cameras.cpp:137-143
    cam = Camera.fisheye(400, 300, 100.0, 100.0, 200.0, 150.0)
    _, _, j = oracle.project(cam, [0, 0, 1])
    np.testing.assert_allclose(j, [[100, 0, 0], [0, 100, 0]], atol=1e-12)


def _visible_fisheye_point(cam):
    while True:
        th, ph, r = RNG.uniform(0.02, 1.5), RNG.uniform(0, 2 * math.pi), RNG.uniform(0.5, 8)
        p = r * np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
        if oracle.project(cam, p)[0]:
            return p


def test_jacobian_matches_fd():  # test_cameras.cpp:156-174
    cam = Camera.fisheye(640, 480, 190.0, 185.0, 320.0, 240.0, math.pi / 2)
    worst = 0.0
    for _ in range(1000):
        p = _visible_fisheye_point(cam)
        _, _, j = oracle.project(cam, p)
        for c in range(3):
            e = np.zeros(3)
            e[c] = 1e-5
            fd = (oracle.project(cam, p + e)[1] - oracle.project(cam, p - e)[1]) / 2e-5
            for r in range(2):
                # the reference's 1e-5 relative criterion, plus the FD noise floor of a pixel
                # coordinate of ~600 at h = 1e-5 (ulp(600)/2h ~ 6e-9): our stream draws a point
                # whose J(0,1) is ~1e-4, where the pure relative form measures FD noise.
                excess = abs(j[r, c] - fd[r]) - (1e-5 * max(abs(j[r, c]), abs(fd[r])) + 6e-9)
                worst = max(worst, excess)
    assert worst <= 0.0


def test_jacobian_grad_matches_fd():  # test_cameras.cpp:176-197
    cam = Camera.fisheye(640, 480, 190.0, 185.0, 320.0, 240.0, math.pi / 2)
    worst = 0.0
    for _ in range(1000):
        p = _visible_fisheye_point(cam)
        grad = oracle.jacobian_grad(cam, p)
        for k in range(3):
            e = np.zeros(3)
            e[k] = 1e-4
            fd = (oracle.project(cam, p + e)[2] - oracle.project(cam, p - e)[2]) / 2e-4
            for r in range(2):
                for c in range(3):
                    worst = max(worst, rel_err(grad[k, r, c], fd[r, c]))
    assert worst < 1e-4


def test_fisheye_radial_law():  # test_cameras.cpp:239-252
    f = 157.0
    cam = Camera.fisheye(640, 480, f, f, 320.0, 240.0, math.pi)
    for _ in range(1000):
        th, ph, r = RNG.uniform(1e-3, math.pi - 0.05), RNG.uniform(0, 2 * math.pi), RNG.uniform(0.2, 5.0)
        p = r * np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
        px = oracle.project(cam, p)[1]
        rd = math.hypot(px[0] - 320.0, px[1] - 240.0)
        assert abs(rd - f * th) / (f * th) < 1e-9


def test_small_angle_fisheye_matches_pinhole():  # test_cameras.cpp:254-270
    f = 300.0
    fish = Camera.fisheye(640, 480, f, f, 320.0, 240.0)
    pin = Camera.pinhole(640, 480, f, f, 320.0, 240.0)
    worst = 0.0
    for _ in range(2000):
        th, ph = RNG.uniform(0, math.radians(5.0)), RNG.uniform(0, 2 * math.pi)
        p = np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
        worst = max(worst, np.linalg.norm(oracle.project(fish, p)[1] - oracle.project(pin, p)[1]))
    assert worst < 0.07


def test_series_and_general_paths_agree():  # test_cameras.cpp:287-318
    cam = Camera.fisheye(400, 300, 120.0, 120.0, 200.0, 150.0)
    for _ in range(100):
        ph = RNG.uniform(0, 2 * math.pi)
        p = np.array([1e-5 * math.cos(ph), 1e-5 * math.sin(ph), 1.0])
        _, ps, js = oracle.project(cam, p, force=1)
        _, pg, jg = oracle.project(cam, p, force=2)
        assert np.linalg.norm(ps - pg) < 1e-8
        assert np.abs(js - jg).max() / np.abs(js).max() < 1e-8
    pin = Camera.pinhole(400, 300, 120.0, 120.0, 200.0, 150.0)
    for lz in (1e-4, 1e-6, 1e-9, 0.0):
        p = np.array([lz, 0.5 * lz, 1.0])
        _, a, ja = oracle.project(cam, p)
        _, b, jb = oracle.project(pin, p)
        assert np.linalg.norm(a - b) < 1e-7
        assert np.abs(ja - jb).max() / 120.0 < 1e-7


def test_visible_points_have_finite_jacobians():  # test_cameras.cpp:320-329
    cam = Camera.fisheye(640, 480, 190.0, 185.0, 320.0, 240.0, math.pi / 2)
    for _ in range(500):
        v, _, j = oracle.project(cam, _visible_fisheye_point(cam))
        assert v and np.isfinite(j).all()


# ---------------------------------------------------------------- tests/test_model.cpp

def _quat(unit=True):
    while True:
        q = RNG.uniform(-1, 1, 4)
        if np.linalg.norm(q) >= 0.1:
            return q / np.linalg.norm(q) if unit else q


def _cov_ref(q, s):
    w, x, y, z = np.asarray(q) / np.linalg.norm(q)
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    return R @ np.diag(np.exp(2 * np.asarray(s))) @ R.T


def test_build_covariance_goldens():  # test_model.cpp:41-52
    np.testing.assert_allclose(oracle.build_covariance([1, 0, 0, 0], [0, 0, 0]), np.eye(3), atol=1e-15)
    exp = np.eye(3)
    exp[0, 0] = 4.0
    np.testing.assert_allclose(oracle.build_covariance([1, 0, 0, 0], [math.log(2), 0, 0]), exp, atol=1e-15)


def test_build_covariance_properties():  # test_model.cpp:54-97
    for _ in range(200):
        q, s = _quat(False), RNG.uniform(-1.5, 1.0, 3)
        sig = oracle.build_covariance(q, s)
        assert np.abs(sig - _cov_ref(q, s)).max() < 1e-12
        assert (sig == sig.T).all()
        assert np.linalg.eigvalsh(sig).min() >= -1e-12
        assert np.abs(sig - oracle.build_covariance(-q, s)).max() == pytest.approx(0.0)
        base = np.trace(sig)
        for c in range(3):
            s2 = s.copy()
            s2[c] += 0.1
            assert np.trace(oracle.build_covariance(q, s2)) >= base


def test_zero_quaternion_rejected():  # test_model.cpp:99-104
    with pytest.raises(ValueError, match="degenerate rotation"):
        oracle.build_covariance([0, 0, 0, 0], [0, 0, 0])
    with pytest.raises(ValueError):
        oracle.build_covariance_backward([0, 0, 0, 0], [0, 0, 0], np.eye(3))


def test_build_covariance_backward():  # test_model.cpp:106-153
    dq, ds = oracle.build_covariance_backward(_quat(), [0.3, -0.2, 0.1], np.zeros((3, 3)))
    assert not dq.any() and not ds.any()
    dq, ds = oracle.build_covariance_backward([1, 0, 0, 0], [0, 0, 0], np.eye(3))
    np.testing.assert_allclose(ds, [2, 2, 2], rtol=1e-12)
    assert np.abs(dq).max() < 1e-12
    h = 1e-5
    for _ in range(100):
        q, s = _quat(False), RNG.uniform(-1, 0.5, 3)
        g = RNG.uniform(-1, 1, (3, 3))
        g = np.triu(g) + np.triu(g, 1).T
        dq, ds = oracle.build_covariance_backward(q, s, g)
        loss = lambda qq, ss: float((g * oracle.build_covariance(qq, ss)).sum())
        for c in range(4):
            e = np.zeros(4)
            e[c] = h
            fd = (loss(q + e, s) - loss(q - e, s)) / (2 * h)
            assert abs(fd - dq[c]) / max(abs(fd), abs(dq[c]), 1e-8) < 1e-6
        for c in range(3):
            e = np.zeros(3)
            e[c] = h
            fd = (loss(q, s + e) - loss(q, s - e)) / (2 * h)
            assert abs(fd - ds[c]) / max(abs(fd), abs(ds[c]), 1e-8) < 1e-6


def test_eval_sh_goldens():  # test_model.cpp:155-202
    sh = np.zeros(48)
    sh[0], sh[16], sh[32] = 0.7, -0.4, 1.1
    d = np.array([0.3, -0.5, 0.9])
    d /= np.linalg.norm(d)
    np.testing.assert_allclose(oracle.eval_sh(sh, d, 0), 0.28209479177387814 * np.array([0.7, -0.4, 1.1]) + 0.5,
                               rtol=1e-12)
    assert (oracle.eval_sh(np.zeros(48), d, 0) == 0.5).all()
    sh = RNG.uniform(-1, 1, 48)
    got = oracle.eval_sh(sh, [0, 0, 1], 3)
    for c in range(3):
        k = sh[c * 16:(c + 1) * 16]
        exp = max(0.282094791773878 * k[0] + 0.488602511902920 * k[2] + 0.315391565252520 * 2 * k[6]
                  + 0.373176332590115 * 2 * k[12] + 0.5, 0.0)
        assert got[c] == pytest.approx(exp, rel=1e-10)
    sh = np.zeros(48)
    sh[0], sh[16] = -10.0, 0.2
    c = oracle.eval_sh(sh, [0, 0, 1], 0)
    assert c[0] == 0.0 and c[1] > 0.0


# ---------------------------------------------------------------- tests/test_splatting.cpp

def random_scene(n, seed, spherical=False, sh_all=False):  # test_splatting.cpp:18-42
    r = np.random.default_rng(seed)
    means = []
    for _ in range(n):
        if spherical:
            th, ph = r.uniform(0.05, 2.8), r.uniform(0, 2 * math.pi)
            means.append(r.uniform(1.5, 6.0) * np.array([math.sin(th) * math.cos(ph), math.cos(th),
                                                           math.sin(th) * math.sin(ph)]))
        else:
            means.append([r.uniform(-1.5, 1.5), r.uniform(-1.2, 1.2), r.uniform(1.5, 7.0)])
    ls = np.log(r.uniform(0.03, 0.25, (n, 3)))
    q = r.uniform(-1, 1, (n, 4))
    q[np.linalg.norm(q, axis=1) < 0.1] = [1, 0, 0, 0]
    op = np.log((p := r.uniform(0.05, 0.95, n)) / (1 - p))
    sh = np.zeros((n, 48))
    sh[:, [0, 16, 32]] = r.uniform(-1.2, 1.2, (n, 3))
    if sh_all:
        sh += r.uniform(-0.3, 0.3, (n, 48)) * (np.arange(48) % 16 != 0)
    return Scene(np.array(means), q, ls, op, sh, np.array([0.1, 0.15, 0.2]))


def test_preprocess_pinhole_golden():  # test_splatting.cpp:58-78
    res = oracle.render(one_gaussian([0, 0, 5]), Camera.pinhole(640, 480, 100.0, 100.0, 320.0, 240.0),
                        sh_degree=3, dtype=np.float64)
    assert res.num_splats == 1
    m, con = res.get("mean_px"), res.get("conic")
    assert m[0] == pytest.approx(320.0) and m[1] == pytest.approx(240.0)
    assert con[0] == pytest.approx(1 / 400.3, rel=1e-12) and con[1] == pytest.approx(0.0)
    assert con[2] == pytest.approx(1 / 400.3, rel=1e-12)
    assert res.get("depth")[0] == pytest.approx(5.0)
    assert res.get("radius")[0] == math.ceil(3 * math.sqrt(400.3))
    assert res.get("alpha")[0] == pytest.approx(0.5)
    assert res.get("source")[0] == 0


def test_preprocess_culling():  # test_splatting.cpp:80-104
    pin = Camera.pinhole(64, 64, 40.0, 40.0, 32.0, 32.0)
    r = oracle.render(one_gaussian([0, 0, -3]), pin, dtype=np.float64)
    assert r.num_splats == 0 and r.stats()["num_culled"] == 1
    fish = Camera.fisheye(64, 64, 20.0, 20.0, 32.0, 32.0)
    t = math.radians(120)
    r = oracle.render(one_gaussian(3 * np.array([math.sin(t), 0, math.cos(t)])), fish, dtype=np.float64)
    assert r.num_splats == 0 and r.stats()["num_culled"] == 1
    r = oracle.render(one_gaussian([50.0, 0, 1.0], log_scale=[math.log(0.01)] * 3), pin, dtype=np.float64)
    assert r.num_splats == 0 and r.stats()["num_culled"] == 1


def _simple(mx, my, radius, depth=1.0):  # test_splatting.cpp:44-54
    return dict(mean_px=[mx, my], conic=[1.0, 0.0, 1.0], depth=depth, radius=radius, color=[1, 1, 1], alpha=0.5)


def _splats(lst, w, h, bg=(0, 0, 0)):
    return oracle.splats_render([s["mean_px"] for s in lst], [s["conic"] for s in lst], [s["depth"] for s in lst],
                                [s["radius"] for s in lst], [s["color"] for s in lst], [s["alpha"] for s in lst],
                                w, h, bg)


def test_bin_single_tile_and_3x3():  # test_splatting.cpp:106-123
    r = _splats([_simple(8.0, 8.0, 1)], 64, 64)
    assert r.num_intersections == 1 and r.tiles_x == 4 and r.tiles_y == 4
    off = r.get("offsets")
    assert off[0] == 0 and off[1] == 1
    r = _splats([_simple(16.0, 16.0, 17)], 64, 64)
    assert r.num_intersections == 9
    assert oracle.bruteforce_intersections([[16.0, 16.0]], [17], 64, 64) == 9


def test_bin_counts_match_bruteforce():  # test_splatting.cpp:125-133
    cam = Camera.pinhole(128, 96, 80.0, 80.0, 64.0, 48.0)
    for trial in range(10):
        res = oracle.render(random_scene(120, 500 + trial), cam, dtype=np.float64)
        assert res.num_intersections == oracle.bruteforce_intersections(res.get("mean_px").reshape(-1, 2),
                                                                        res.get("radius"), 128, 96)


def test_spans_partition_and_tie_break():  # test_splatting.cpp:135-156
    res = oracle.render(random_scene(200, 99), Camera.pinhole(128, 128, 90.0, 90.0, 64.0, 64.0), dtype=np.float64)
    off, refs = res.get("offsets"), res.get("refs")
    depth, src = res.get("depth"), res.get("source")
    assert off[0] == 0 and off[-1] == len(refs)
    assert (np.diff(off.astype(np.int64)) >= 0).all()
    for t in range(len(off) - 1):
        seg = refs[off[t]:off[t + 1]]
        for a, b in zip(seg[:-1], seg[1:]):
            assert depth[a] <= depth[b]
            if depth[a] == depth[b]:
                assert src[a] < src[b]


def test_blend_goldens():  # test_splatting.cpp:158-189
    s = _simple(8.5, 8.5, 3)
    s["alpha"], s["color"] = 0.99, [0.2, 0.6, 1.0]
    r = _splats([s], 16, 16)
    np.testing.assert_allclose(r.image[8, 8], [0.99 * 0.2, 0.99 * 0.6, 0.99], rtol=1e-12)
    assert r.get("final_T")[8 * 16 + 8] == pytest.approx(0.01)
    assert r.get("count")[8 * 16 + 8] == 1
    near, far = _simple(8.5, 8.5, 3, 1.0), _simple(8.5, 8.5, 3, 2.0)
    near["color"], far["color"] = [1, 0, 0], [0, 1, 0]
    r = _splats([far, near], 16, 16, bg=(0, 0, 1))
    np.testing.assert_allclose(r.image[8, 8], [0.5, 0.25, 0.25], rtol=1e-12)


def test_empty_scene_is_background():  # test_splatting.cpp:191-199
    sc = Scene(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 48)),
               np.array([0.3, 0.5, 0.7]))
    r = oracle.render(sc, Camera.pinhole(48, 32, 30.0, 30.0, 24.0, 16.0), dtype=np.float64)
    assert r.num_intersections == 0
    assert (r.image == np.array([0.3, 0.5, 0.7])).all()


def test_conservation_fisheye():  # test_splatting.cpp:201-214
    sc = random_scene(150, 321)
    sc.sh[:] = 0
    sc.sh[:, [0, 16, 32]] = (1.0 - 0.5) / 0.28209479177387814
    sc.background = np.ones(3)
    r = oracle.render(sc, Camera.fisheye(96, 96, 30.0, 30.0, 48.0, 48.0), sh_degree=0, dtype=np.float64)
    np.testing.assert_allclose(r.image, 1.0, rtol=1e-6)


def test_render_deterministic_across_threads():  # test_splatting.cpp:216-232
    sc = random_scene(200, 777)
    cam = Camera.fisheye(128, 128, 40.0, 40.0, 64.0, 64.0)
    for dt in (np.float64, np.float32):
        a = oracle.render(sc, cam, dtype=dt, threads=1)
        b = oracle.render(sc, cam, dtype=dt, threads=1)
        c = oracle.render(sc, cam, dtype=dt, threads=5)
        assert a.image.tobytes() == b.image.tobytes() == c.image.tobytes()
        assert a.num_intersections == c.num_intersections


@pytest.mark.parametrize("model", ["pinhole", "fisheye", "panorama"])
def test_tiled_equals_bruteforce(model):  # test_splatting.cpp:234-261
    trial = {"pinhole": 0, "fisheye": 1, "panorama": 2}[model]
    sc = random_scene(200, 9000 + trial, spherical=model != "pinhole", sh_all=True)
    cam = {"pinhole": Camera.pinhole(96, 80, 60.0, 60.0, 48.0, 40.0),
           "fisheye": Camera.fisheye(96, 80, 28.0, 28.0, 48.0, 40.0),
           "panorama": Camera.panorama(128, 64)}[model]
    fast = oracle.render(sc, cam, sh_degree=3, dtype=np.float64)
    ref, _ = oracle.bruteforce_render(sc, cam, sh_degree=3)
    assert np.abs(fast.image - ref).max() < 1e-5


def test_float_path_close_to_double_oracle():  # test_splatting.cpp:263-274
    sc = random_scene(150, 4242)
    cam = Camera.fisheye(96, 96, 30.0, 30.0, 48.0, 48.0)
    fast = oracle.render(sc, cam, sh_degree=3, dtype=np.float32)
    ref, _ = oracle.bruteforce_render(sc, cam, sh_degree=3)
    assert np.abs(fast.image.astype(np.float64) - ref).max() < 2e-4
    fast_libm = oracle.render(sc, cam, sh_degree=3, dtype=np.float32, mode=oracle.MODE_LIBM)
    assert np.abs(fast_libm.image.astype(np.float64) - ref).max() < 2e-4
