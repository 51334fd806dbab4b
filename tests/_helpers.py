"""Shared helpers for the parity tests (oracle side and GPU side)."""
from __future__ import annotations

import numpy as np

from paper_2409_04751_b200 import Camera, Scene, synthetic


def to_device(scene: Scene, device="cuda"):
    import torch

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)
    return Scene(t(scene.means), t(scene.rotations), t(scene.log_scales), t(scene.opacity_logits), t(scene.sh),
                 np.asarray(scene.background, np.float32))


def psnr(a, b, peak=1.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10 * np.log10(peak * peak / mse)


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


GROUPS = {"mean": slice(0, 3), "rotation": slice(3, 7), "log_scale": slice(7, 10), "opacity": slice(10, 11),
          "sh_dc": [11, 27, 43], "sh_rest": [c * 16 + j + 11 for c in range(3) for j in range(1, 16)]}


def small_fisheye(w=256, h=192, fov=np.pi / 2):
    f = 0.5 * np.hypot(w, h) / fov
    return Camera.fisheye(w, h, f, f, w / 2, h / 2, fov).as_float32()


def config_case(idx, n, seed_shift=0):
    scene, deg, cams, dls = synthetic.config(idx, n=n)
    return scene, deg, cams, dls
