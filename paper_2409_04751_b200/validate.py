"""Large-scene validation on the GPU.

  bruteforce_render  inc/oracle.hpp:161-270 -- the reference's brute-force renderer in double on
                     the GPU (fgs_bruteforce_render[_f64]): independent projection / covariance /
                     SH code, global (depth, source) order, every splat gated per tile. Usable at
                     the configs' full scale, where the CPU brute force (O(N x P)) is not.
  gradcheck          inc/oracle.hpp:338-418 -- analytic gradients of L = sum(image^2) from the
                     fast path's backward against central finite differences of the brute-force
                     renderer's loss (double scene perturbations), per parameter group, with the
                     reference's report format (GradcheckReport::to_lines, :300-318).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _lib
from .api import Rasterizer, _camera_struct
from .types import BackwardOptions, Camera, RenderOptions, Scene


def _dev(a, dtype):
    import torch

    return torch.as_tensor(np.ascontiguousarray(np.asarray(a), dtype)).cuda()


def bruteforce_render(rast: Rasterizer, scene: Scene, camera: Camera, sh_degree: int = 0, background=None,
                      double_scene: bool = False, want_transmittance: bool = False):
    """Image (H, W, 3) float64 numpy (and transmittance (H, W)) of the brute-force renderer.
    ``scene`` holds host arrays; ``double_scene`` keeps them in double on the device."""
    import torch

    bg = np.asarray(scene.background if background is None else background, np.float64).reshape(3)
    bgc = (C.c_double * 3)(*bg)
    cam = _camera_struct(camera)
    img = torch.empty((camera.height, camera.width, 3), dtype=torch.float64, device="cuda")
    tr = torch.empty((camera.height, camera.width), dtype=torch.float64, device="cuda") if want_transmittance else None
    trp = C.c_void_p(tr.data_ptr()) if tr is not None else None
    if double_scene:
        arrs = [_dev(getattr(scene, f), np.float64) for f in ("means", "rotations", "log_scales", "opacity_logits",
                                                              "sh")]
        rc = rast._L.fgs_bruteforce_render_f64(rast._h, scene.n, *[C.c_void_p(a.data_ptr()) for a in arrs],
                                               C.byref(cam), int(sh_degree), bgc, C.c_void_p(img.data_ptr()), trp)
    else:
        arrs = [_dev(getattr(scene, f), np.float32) for f in ("means", "rotations", "log_scales", "opacity_logits",
                                                              "sh")]
        g = _lib.fgs_gaussians()
        g.n = scene.n
        g.means, g.rotations, g.log_scales, g.opacity_logits, g.sh = [a.data_ptr() for a in arrs]
        rc = rast._L.fgs_bruteforce_render(rast._h, C.byref(g), C.byref(cam), int(sh_degree), bgc,
                                           C.c_void_p(img.data_ptr()), trp)
    rast._check(rc)
    out = img.cpu().numpy()
    return (out, tr.cpu().numpy()) if want_transmittance else out


@dataclass
class GradcheckGroup:  # oracle.hpp:292-298
    name: str
    max_rel_err: float = 0.0
    worst_gaussian: int = -1
    worst_component: int = -1
    passed: bool = True


@dataclass
class GradcheckReport:  # oracle.hpp:300-318
    groups: List[GradcheckGroup] = field(default_factory=list)
    tolerance: float = 1e-3
    passed: bool = True

    def to_lines(self) -> str:
        out = [f"group={g.name} max_rel_err={g.max_rel_err:g} worst_gaussian={g.worst_gaussian} "
               f"worst_component={g.worst_component} pass={1 if g.passed else 0}" for g in self.groups]
        out.append(f"overall tolerance={self.tolerance:g} pass={1 if self.passed else 0}")
        return "\n".join(out) + "\n"


def relative_error(a, b):  # oracle.hpp:37-40
    return abs(a - b) / max(abs(a), abs(b), 1e-8)


GROUPS = (("mean", 0, 3), ("rotation", 3, 4), ("log_scale", 7, 3), ("opacity", 10, 1), ("sh_dc", 11, 3))


def gradcheck(rast: Rasterizer, scene: Scene, camera: Camera, step: float = 1e-4, tolerance: float = 1e-3,
              jacobian_grad_scale=(1.0, 1.0, 1.0)) -> GradcheckReport:
    """oracle.hpp:338-418 with the B200 path as the analytic side (SH degree 0, L = sum image^2):
    14 parameters per Gaussian (mean 3, rotation 4, log-scale 3, opacity 1, SH DC 3)."""
    import torch
    from .api import grads_as_rows

    sc32 = scene.astype(np.float32)
    ds = Scene(*[_dev(getattr(sc32, f), np.float32) for f in ("means", "rotations", "log_scales", "opacity_logits",
                                                              "sh")], np.asarray(scene.background, np.float32))
    cam32 = camera.as_float32()
    img, _ = rast.forward(ds, cam32, RenderOptions(sh_degree=0, background=scene.background))
    g = rast.backward(ds, cam32, 2.0 * img, BackwardOptions(full_sh=False, jacobian_grad_scale=jacobian_grad_scale))
    torch.cuda.synchronize()
    analytic = grads_as_rows(g, scene.n).astype(np.float64)
    base = scene.astype(np.float64)
    n = scene.n
    fd = np.zeros((n, 14))

    def loss(sc):
        return float(np.sum(bruteforce_render(rast, sc, cam32, 0, double_scene=True) ** 2))

    fields = [("means", 3), ("rotations", 4), ("log_scales", 3), ("opacity_logits", 1)]
    for gi in range(n):
        for p in range(14):
            vals = []
            for delta in (step, -step):
                sc = Scene(base.means.copy(), base.rotations.copy(), base.log_scales.copy(),
                           base.opacity_logits.copy(), base.sh.copy(), base.background)
                if p < 11:
                    off = 0
                    for name, w in fields:
                        if p < off + w:
                            arr = getattr(sc, name)
                            if arr.ndim == 1:
                                arr[gi] += delta
                            else:
                                arr[gi, p - off] += delta
                            break
                        off += w
                else:
                    sc.sh[gi, (p - 11) * 16] += delta
                vals.append(loss(sc))
            fd[gi, p] = (vals[0] - vals[1]) / (2.0 * step)
    cols = list(range(11)) + [11, 27, 43]  # analytic rows: sh DC at 11 + 16c
    a14 = analytic[:, cols]
    rep = GradcheckReport(tolerance=tolerance)
    for name, start, width in GROUPS:
        grp = GradcheckGroup(name)
        for gi in range(n):
            for c in range(width):
                err = relative_error(a14[gi, start + c], fd[gi, start + c])
                if err > grp.max_rel_err:
                    grp.max_rel_err, grp.worst_gaussian, grp.worst_component = err, gi, c
        grp.passed = grp.max_rel_err < tolerance
        rep.passed = rep.passed and grp.passed
        rep.groups.append(grp)
    return rep
