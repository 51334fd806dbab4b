"""Plain data types mirroring the reference's scene / camera / options structs.

Reference: /root/reference/proj/include/omnisplat/
  - Gaussian3D / Scene           model.hpp:18-51
  - Camera (+ fisheye factory)   cameras.hpp:29-74
  - RenderOptions                splatting.hpp:50-55
  - RenderStats                  splatting.hpp:41-48
  - BackwardOptions              gradients.hpp:57-63

The scene is stored structure-of-arrays (one contiguous array per field), which is the
layout the C ABI (include/fgs.h) takes. SH coefficients keep the reference's in-memory
order: per Gaussian, 48 floats indexed ``channel * 16 + basis`` (Eigen column-major
``Matrix<S, 16, 3>``, core.hpp:23).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

CAMERA_PINHOLE = 0
CAMERA_FISHEYE = 1
CAMERA_PANORAMA = 2

GRAD_STRIDE = 59  # mean 3, rotation 4, log_scale 3, opacity 1, sh 48
GRAD_SLICES = {
    "mean": slice(0, 3),
    "rotation": slice(3, 7),
    "log_scale": slice(7, 10),
    "opacity": slice(10, 11),
    "sh": slice(11, 59),
}


@dataclass
class Camera:
    """Camera (cameras.hpp:29-74): equidistant fisheye (the paper's model), pinhole or
    equirectangular panorama -- all three on the B200 path (only K1/K4b differ)."""

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    rotation_wc: np.ndarray = field(default_factory=lambda: np.eye(3))  # world -> camera
    translation_wc: np.ndarray = field(default_factory=lambda: np.zeros(3))
    fov_max: float = math.pi / 2
    model: int = CAMERA_FISHEYE

    @staticmethod
    def fisheye(w, h, fx, fy, cx, cy, fov_max=math.pi / 2) -> "Camera":
        return Camera(w, h, fx, fy, cx, cy, fov_max=fov_max, model=CAMERA_FISHEYE)

    @staticmethod
    def pinhole(w, h, fx, fy, cx, cy) -> "Camera":
        return Camera(w, h, fx, fy, cx, cy, model=CAMERA_PINHOLE)

    @staticmethod
    def panorama(w, h) -> "Camera":
        return Camera(w, h, 0.0, 0.0, 0.0, 0.0, model=CAMERA_PANORAMA)

    def as_float32(self) -> "Camera":
        """The camera as the fp32 path sees it (every field rounded to float)."""
        f = lambda v: float(np.float32(v))
        return Camera(self.width, self.height, f(self.fx), f(self.fy), f(self.cx), f(self.cy),
                      np.asarray(self.rotation_wc, np.float32).astype(np.float64),
                      np.asarray(self.translation_wc, np.float32).astype(np.float64),
                      f(self.fov_max), self.model)

    def to_array(self) -> np.ndarray:
        """[model, w, h, fx, fy, cx, cy, R(9 row-major), t(3), fov_max] as float64."""
        a = np.zeros(20, np.float64)
        a[0], a[1], a[2] = self.model, self.width, self.height
        a[3:7] = (self.fx, self.fy, self.cx, self.cy)
        a[7:16] = np.asarray(self.rotation_wc, np.float64).reshape(9)
        a[16:19] = np.asarray(self.translation_wc, np.float64).reshape(3)
        a[19] = self.fov_max
        return a

    def same_as(self, other: "Camera") -> bool:
        """The reference's context/camera equality check (gradients.hpp:213-218)."""
        return (self.model == other.model and self.width == other.width and self.height == other.height
                and self.fx == other.fx and self.fy == other.fy and self.cx == other.cx
                and self.cy == other.cy
                and np.array_equal(np.asarray(self.rotation_wc), np.asarray(other.rotation_wc))
                and np.array_equal(np.asarray(self.translation_wc), np.asarray(other.translation_wc)))

    @property
    def tiles_x(self) -> int:
        return (self.width + 15) // 16

    @property
    def tiles_y(self) -> int:
        return (self.height + 15) // 16


@dataclass
class Scene:
    """Structure-of-arrays Gaussian scene (model.hpp:18-51). Arrays may be numpy (host) or
    torch tensors (host or CUDA); shapes: means (N,3), rotations (N,4) w,x,y,z unnormalised,
    log_scales (N,3), opacity_logits (N,), sh (N,48) [channel*16 + basis]."""

    means: object
    rotations: object
    log_scales: object
    opacity_logits: object
    sh: object
    background: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    def astype(self, dtype) -> "Scene":
        c = lambda a: np.ascontiguousarray(np.asarray(a), dtype=dtype)
        return Scene(c(self.means), c(self.rotations), c(self.log_scales), c(self.opacity_logits),
                     c(self.sh), np.asarray(self.background, dtype=dtype))

    def subset(self, idx) -> "Scene":
        return Scene(self.means[idx], self.rotations[idx], self.log_scales[idx],
                     self.opacity_logits[idx], self.sh[idx], self.background)


@dataclass
class RenderOptions:
    """splatting.hpp:50-55. ``background`` overrides the scene background when given."""

    sh_degree: int = 3
    background: Optional[np.ndarray] = None


@dataclass
class RenderStats:
    """splatting.hpp:41-48 (stage times measured with CUDA events on the GPU path)."""

    num_intersections: int = 0
    num_splats: int = 0
    num_culled: int = 0
    num_degenerate: int = 0
    preprocess_ms: float = 0.0
    binning_ms: float = 0.0
    sort_ms: float = 0.0
    raster_ms: float = 0.0
    peak_aux_bytes: int = 0


@dataclass
class BackwardOptions:
    """gradients.hpp:57-63 plus the B200 build's SH switch.

    ``jacobian_grad_scale`` is the reference's mutation hook. ``full_sh`` (default on)
    returns all 48 SH gradients; off reproduces the reference's DC-only buffer.
    ``sh_view_dir_grad`` (default off, for reference parity) adds the colour -> view-direction
    -> mean term the reference omits (gradients.hpp:255-262).
    """

    jacobian_grad_scale: tuple = (1.0, 1.0, 1.0)
    full_sh: bool = True
    sh_view_dir_grad: bool = False
