"""Training step around the rasterizer: the reference's loss, optimizer
and train loop, with the loss, backward and Adam update on the device.

Reference (omnisplat, /root/reference/proj/include/omnisplat/):
  l1_dssim_loss  metrics.hpp:172-195 (ssim :86-161)   -> ``l1_dssim_loss`` (fgs_l1_dssim_loss)
  adam_step      optimize.hpp:100-145                  -> ``Trainer.adam_step`` (fgs_adam_step)
  TrainConfig / GroupLearningRates / camera_extent     optimize.hpp:56-97, :148-160
  train          optimize.hpp:190-277                  -> ``train`` (fgs_train_step per iteration)

The device path is fp32 (the reference trains in double); the loss and gradient agree within
the tolerances the GPU tests state. ``lr_sh_rest`` (SH bands 1..3) is a build extension: the
reference optimises the DC coefficients only, and 0 (the default) reproduces that.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from .api import FgsError, InvalidArgument, Rasterizer, _camera_struct
from .types import Camera, Scene


class NonFinite(RuntimeError):
    """std::runtime_error from adam_step / train (non-finite gradient or loss)."""


@dataclass
class TrainConfig:  # optimize.hpp:56-70
    iterations: int = 2000
    lr_mean: float = 1.6e-4  # scaled by the camera extent at train time
    lr_rotation: float = 1e-3
    lr_log_scale: float = 5e-3
    lr_opacity: float = 5e-2
    lr_sh_dc: float = 2.5e-3
    lr_sh_rest: float = 0.0
    loss_lambda: float = 0.2
    random_background: bool = False
    seed: int = 0
    sh_degree: int = 0
    eval_every: int = 100


@dataclass
class View:  # optimize.hpp:26-32
    camera: Camera
    image: np.ndarray  # H x W x 3
    transmittance: Optional[np.ndarray] = None  # H x W


@dataclass
class Dataset:  # optimize.hpp:34-54
    views: List[View]
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @staticmethod
    def is_test_view(i):
        return i % 8 == 0

    def train_indices(self):
        return [i for i in range(len(self.views)) if not self.is_test_view(i)]

    def test_indices(self):
        return [i for i in range(len(self.views)) if self.is_test_view(i)]


def camera_center(cam: Camera) -> np.ndarray:
    r = np.asarray(cam.rotation_wc, np.float64)
    return -r.T @ np.asarray(cam.translation_wc, np.float64)


def camera_extent(dataset: Dataset) -> float:
    """optimize.hpp:148-160: 1.1 x the camera rig's radius (1 if degenerate)."""
    if not dataset.views:
        return 1.0
    c = np.array([camera_center(v.camera) for v in dataset.views])
    radius = float(np.max(np.linalg.norm(c - c.mean(axis=0), axis=1)))
    return 1.1 * radius if radius > 0 else 1.0


def _check(L, h, rc):
    if rc == _lib.FGS_OK:
        return
    msg = L.fgs_last_error(h).decode()
    if rc == _lib.FGS_ENONFINITE:
        raise NonFinite(msg)
    if rc in (_lib.FGS_EINVAL, _lib.FGS_EDEGENERATE_QUAT):
        raise InvalidArgument(msg)
    raise FgsError(f"status {rc}: {msg}")


def l1_dssim_loss(rast: Rasterizer, rendered, target, lam: float = 0.2):
    """(total, l1, dssim, d_rendered) for device tensors rendered/target (H x W x 3 fp32)."""
    import torch

    if tuple(rendered.shape) != tuple(target.shape):
        raise InvalidArgument("l1_dssim_loss: image dimensions differ")
    h, w = int(rendered.shape[0]), int(rendered.shape[1])
    d = torch.empty_like(rendered)
    out = (C.c_double * 3)()
    _check(rast._L, rast._h, rast._L.fgs_l1_dssim_loss(rast._h, C.c_void_p(rendered.data_ptr()),
                                                       C.c_void_p(target.data_ptr()), w, h, float(lam),
                                                       C.c_void_p(d.data_ptr()), out))
    return out[0], out[1], out[2], d


def _grads_struct(buf, n):
    g = _lib.fgs_gradients()
    base = buf.data_ptr()
    off = 0
    for name, width in (("d_means", 3), ("d_rotations", 4), ("d_log_scales", 3), ("d_opacity_logits", 1),
                        ("d_sh", 48)):
        setattr(g, name, base + 4 * off)
        off += width * n
    return g


class Trainer:
    """Device-resident scene + Adam state (AdamState, optimize.hpp:78-90). The scene's five
    parameter arrays live in one 59*N fp32 buffer (field blocks, the gradient layout)."""

    def __init__(self, scene: Scene, config: TrainConfig = None, extent: float = 1.0, device: int = 0,
                 rasterizer: Optional[Rasterizer] = None):
        import torch

        self.cfg = config or TrainConfig()
        self.rast = rasterizer or Rasterizer(device)
        self.n = n = scene.n
        dev = torch.device("cuda", device)
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float32)).reshape(-1)
        self.params = torch.cat([t(scene.means), t(scene.rotations), t(scene.log_scales), t(scene.opacity_logits),
                                 t(scene.sh)]).to(dev)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.background = np.asarray(scene.background, np.float32)
        self.state = _lib.fgs_adam_state()
        self.state.step = 0
        self.state.m = _grads_struct(self.m, n)
        self.state.v = _grads_struct(self.v, n)
        c = self.cfg
        self.adam = _lib.fgs_adam_options(c.lr_mean * extent, c.lr_rotation, c.lr_log_scale, c.lr_opacity,
                                          c.lr_sh_dc, c.lr_sh_rest, 0.9, 0.999, 1e-15)

    @property
    def step_count(self) -> int:
        return int(self.state.step)

    def _params_struct(self):
        g = _grads_struct(self.params, self.n)
        p = _lib.fgs_params()
        p.n = self.n
        p.means, p.rotations, p.log_scales, p.opacity_logits, p.sh = (g.d_means, g.d_rotations, g.d_log_scales,
                                                                      g.d_opacity_logits, g.d_sh)
        return p

    def scene(self, device=True) -> Scene:
        """The current parameters as a Scene (device views, or host copies)."""
        n, p = self.n, self.params
        parts, off = [], 0
        for width in (3, 4, 3, 1, 48):
            a = p[off:off + width * n]
            parts.append(a.reshape(n, width) if width > 1 else a)
            off += width * n
        if not device:
            parts = [a.cpu().numpy() for a in parts]
        return Scene(*parts, self.background.copy())

    def adam_step(self, grads):
        """adam_step on the device with a 59*N gradient buffer in the same field-block layout."""
        p = self._params_struct()
        g = _grads_struct(grads, self.n)
        _check(self.rast._L, self.rast._h, self.rast._L.fgs_adam_step(self.rast._h, C.byref(p), C.byref(g),
                                                                      C.byref(self.state), C.byref(self.adam)))

    def step(self, camera: Camera, target, background=None):
        """One train-loop iteration (optimize.hpp:237-266) on a device target image:
        render, L1 + D-SSIM, backward, Adam. Returns (total, l1, dssim)."""
        p = self._params_struct()
        o = _lib.fgs_train_options()
        o.sh_degree = int(self.cfg.sh_degree)
        bg = self.background if background is None else np.asarray(background, np.float32)
        for k in range(3):
            o.background[k] = float(bg[k])
        o.lam = float(self.cfg.loss_lambda)
        o.adam = self.adam
        out = (C.c_double * 3)()
        cam = _camera_struct(camera)
        _check(self.rast._L, self.rast._h,
               self.rast._L.fgs_train_step(self.rast._h, C.byref(p), C.byref(cam), C.c_void_p(target.data_ptr()),
                                           C.byref(o), C.byref(self.state), out))
        return out[0], out[1], out[2]


@dataclass
class TrainResult:  # optimize.hpp:170-176
    scene: Scene
    trace: list
    test_psnr: float = 0.0


def psnr(a, b) -> float:
    """metrics.hpp:73-83."""
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return 100.0 if mse < 1e-10 else min(100.0, 10.0 * math.log10(1.0 / mse))


def train(initial: Scene, dataset: Dataset, config: TrainConfig, device: int = 0) -> TrainResult:
    """optimize.hpp:190-277: cycle shuffled training views, render, L1 + D-SSIM, backward,
    Adam; evaluate test PSNR every eval_every iterations. (The view shuffle uses numpy's
    generator, not std::mt19937_64, so the visiting order differs from the reference's.)"""
    import torch

    train_idx = dataset.train_indices()
    if not train_idx:
        raise InvalidArgument("train: dataset has no training views")
    if config.iterations <= 0:
        raise InvalidArgument("train: iterations must be positive")
    tr = Trainer(initial, config, extent=camera_extent(dataset), device=device)
    rng = np.random.default_rng(config.seed)
    targets = {i: torch.as_tensor(np.ascontiguousarray(dataset.views[i].image, np.float32)).cuda(device)
               for i in range(len(dataset.views))}
    bg0 = np.asarray(dataset.background, np.float32)

    def test_psnr():
        idx = dataset.test_indices()
        if not idx:
            return 0.0
        from .types import RenderOptions

        vals = []
        for i in idx:
            img, _ = tr.rast.forward(tr.scene(), dataset.views[i].camera,
                                     RenderOptions(sh_degree=config.sh_degree, background=bg0))
            vals.append(psnr(img.cpu().numpy(), dataset.views[i].image))
        return float(np.mean(vals))

    order, cursor, trace = list(train_idx), len(train_idx), []
    for it in range(1, config.iterations + 1):
        if cursor >= len(order):
            rng.shuffle(order)
            cursor = 0
        vi = order[cursor]
        cursor += 1
        view = dataset.views[vi]
        bg = bg0
        target = targets[vi]
        if config.random_background:
            bg = rng.uniform(0, 1, 3).astype(np.float32)
            if view.transmittance is not None:
                shift = torch.as_tensor(bg - bg0, device=target.device)
                tt = torch.as_tensor(np.asarray(view.transmittance, np.float32), device=target.device)
                target = target + tt[:, :, None] * shift
        total, _, _ = tr.step(view.camera, target, bg)
        row = {"iteration": it, "loss": total}
        if config.eval_every > 0 and it % config.eval_every == 0:
            row["test_psnr"] = test_psnr()
        trace.append(row)
    return TrainResult(tr.scene(device=False), trace, test_psnr())
