"""Seeded synthetic workloads for BASELINE.json configs 0-4.

The reference measures nothing on a public dataset for this path; the configs are
synthetic. Draw order per config is fixed: means, log-scales, quaternions, opacity
logits, SH, cameras, dL/dpixel, all from ``numpy.random.default_rng(seed)`` with
seed = config index, then cast to fp32.
"""
from __future__ import annotations

import math

import numpy as np

from .types import Camera, Scene

W_FULL, H_FULL = 1752, 1168
HALF_DIAG = 0.5 * math.hypot(W_FULL, H_FULL)


def _unit(rng, n, d):
    v = rng.standard_normal((n, d))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _shell(rng, n, r0, r1):
    r = np.cbrt(rng.uniform(r0 ** 3, r1 ** 3, size=n))
    return _unit(rng, n, 3) * r[:, None]


def _rest(rng, n, means, sh_degree, sh_rest_sigma=0.05):
    log_scales = rng.normal(-4.0, 0.5, size=(n, 3))
    rotations = _unit(rng, n, 4)
    opacity = rng.normal(0.0, 1.0, size=n)
    sh = np.zeros((n, 3, 16))
    sh[:, :, 0] = rng.normal(0.0, 0.3, size=(n, 3))
    if sh_degree > 0:
        sh[:, :, 1:] = rng.normal(0.0, sh_rest_sigma, size=(n, 3, 15))
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return Scene(f(means), f(rotations), f(log_scales), f(opacity), f(sh.reshape(n, 48)),
                 np.zeros(3, np.float32))


def fisheye_full(fov_half=math.pi / 2, rotation_wc=None, translation_wc=None) -> Camera:
    """1752x1168 equidistant fisheye whose half-diagonal maps to ``fov_half``."""
    f = HALF_DIAG / fov_half
    cam = Camera.fisheye(W_FULL, H_FULL, f, f, W_FULL / 2, H_FULL / 2, fov_half)
    if rotation_wc is not None:
        cam.rotation_wc = rotation_wc
        cam.translation_wc = translation_wc
    return cam.as_float32()


def random_pose(rng, box=5.0):
    """Eye ~ U([-box, box]^3), camera-to-world rotation from a uniform random quaternion."""
    eye = rng.uniform(-box, box, size=3)
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    r_cw = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    r_wc = r_cw.T
    return r_wc, -r_wc @ eye


def config(idx: int, n: int | None = None, views: int | None = None, rank: int = 0):
    """Return (scene, sh_degree, cameras[list], dl_dpixel[list or None]) for config ``idx``.

    ``n`` shrinks the Gaussian count (for parity tests); ``views`` overrides the view count
    of configs 3/4; ``rank`` seeds config 4's per-GPU views.
    """
    if idx == 0:
        rng = np.random.default_rng(0)
        n = n or 10_000
        means = _shell(rng, n, 1.0, 10.0)
        scene = _rest(rng, n, means, 0)
        cam = Camera.fisheye(256, 256, 256 / math.pi, 256 / math.pi, 128.0, 128.0).as_float32()
        return scene, 0, [cam], None
    if idx in (1, 2):
        rng = np.random.default_rng(idx)
        if idx == 1:
            n = n or 200_000
            means = _shell(rng, n, 1.0, 10.0)
        else:
            n = n or 1_000_000
            centers = _shell(rng, 64, 2.0, 15.0)
            pick = rng.integers(0, 64, size=n)
            means = centers[pick] + rng.normal(0.0, 0.5, size=(n, 3))
        scene = _rest(rng, n, means, 3)
        cam = fisheye_full()
        dl = rng.standard_normal((H_FULL, W_FULL, 3)).astype(np.float32)
        return scene, 3, [cam], [dl]
    if idx in (3, 4):
        rng = np.random.default_rng(3)
        n = n or 3_000_000
        means = rng.uniform(-10.0, 10.0, size=(n, 3))
        scene = _rest(rng, n, means, 3)
        if idx == 3:
            views = views or 64
            fov = math.radians(95.0)
            cams = [fisheye_full(fov, *random_pose(rng)) for _ in range(views)]
            return scene, 3, cams, None
        views = views or 8
        vr = np.random.default_rng(1000 + rank)
        cams = [fisheye_full(math.pi / 2, *random_pose(vr)) for _ in range(views)]
        dls = [vr.standard_normal((H_FULL, W_FULL, 3)).astype(np.float32) for _ in range(views)]
        return scene, 3, cams, dls
    raise ValueError(f"unknown config {idx}")
