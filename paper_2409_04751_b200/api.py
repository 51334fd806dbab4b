"""Host-side mirror of the reference's render / backward API over the C ABI.

Reference (omnisplat, /root/reference/proj/include/omnisplat/):
  render<S>(scene, camera, options) -> RenderResult{image, stats, context}   splatting.hpp:330-374
  backward<S>(scene, camera, context, dl_dimage, options) -> GradientBuffer  gradients.hpp:207-267
Errors: the reference throws std::invalid_argument (shape / context mismatch, zero quaternion);
here those raise ``InvalidArgument`` (a ValueError) with the reference's messages.

Two entry styles:
  * ``render`` / ``backward`` — host (numpy) arrays in and out, like the reference; the device
    copies happen inside the C ABI's host-buffer calls (fgs_render_host / fgs_backward_host).
  * ``Rasterizer.forward`` / ``.backward`` — device-resident torch CUDA tensors (no copies).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .types import BackwardOptions, Camera, RenderOptions, RenderStats, Scene

GRAD_FIELDS = (("d_means", 3), ("d_rotations", 4), ("d_log_scales", 3), ("d_opacity_logits", 1), ("d_sh", 48))


class InvalidArgument(ValueError):
    """std::invalid_argument analogue."""


class FgsError(RuntimeError):
    pass


def _camera_struct(cam: Camera) -> _lib.fgs_camera:
    c = _lib.fgs_camera()
    c.model = int(cam.model)
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    r = np.asarray(cam.rotation_wc, np.float32).reshape(9)
    t = np.asarray(cam.translation_wc, np.float32).reshape(3)
    for i in range(9):
        c.rotation_wc[i] = float(r[i])
    for i in range(3):
        c.translation_wc[i] = float(t[i])
    c.fov_max = float(cam.fov_max)
    return c


def _render_options(opts: Optional[RenderOptions], scene_bg) -> _lib.fgs_render_options:
    o = _lib.fgs_render_options()
    opts = opts or RenderOptions()
    o.sh_degree = int(opts.sh_degree)
    bg = opts.background if opts.background is not None else scene_bg
    bg = np.zeros(3) if bg is None else np.asarray(bg, np.float64).reshape(3)
    o.use_background = 1
    for k in range(3):
        o.background[k] = float(bg[k])
    return o


def _backward_options(opts: Optional[BackwardOptions], accumulate: bool) -> _lib.fgs_backward_options:
    opts = opts or BackwardOptions()
    o = _lib.fgs_backward_options()
    for k in range(3):
        o.jacobian_grad_scale[k] = float(opts.jacobian_grad_scale[k])
    o.full_sh = 1 if opts.full_sh else 0
    o.accumulate = 1 if accumulate else 0
    o.sh_view_dir_grad = 1 if opts.sh_view_dir_grad else 0
    return o


def _ptr(a) -> int:
    if a is None:
        return 0
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


class Rasterizer:
    """One fgs_context (device, stream, forward state). Not thread-safe, like the C ABI."""

    def __init__(self, device: int = 0):
        self._L = _lib.load()
        self._h = C.c_void_p()
        rc = self._L.fgs_create(int(device), C.byref(self._h))
        if rc != _lib.FGS_OK:
            raise FgsError(f"fgs_create(device={device}) failed with status {rc} (is a CUDA device present?)")
        self.device = device
        self._keep = []

    def close(self):
        if self._h:
            self._L.fgs_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc == _lib.FGS_OK:
            return
        msg = self._L.fgs_last_error(self._h).decode()
        if rc in (_lib.FGS_EINVAL, _lib.FGS_EDEGENERATE_QUAT):
            raise InvalidArgument(msg)
        raise FgsError(f"status {rc}: {msg}")

    def set_stream(self, stream_handle: int):
        self._check(self._L.fgs_set_stream(self._h, C.c_void_p(int(stream_handle))))

    def set_flags(self, flags: int):
        self._check(self._L.fgs_set_flags(self._h, int(flags)))

    @staticmethod
    def _gaussians(scene: Scene) -> _lib.fgs_gaussians:
        g = _lib.fgs_gaussians()
        g.n = scene.n
        g.means, g.rotations, g.log_scales = _ptr(scene.means), _ptr(scene.rotations), _ptr(scene.log_scales)
        g.opacity_logits, g.sh = _ptr(scene.opacity_logits), _ptr(scene.sh)
        return g

    # ---- device-resident path (torch CUDA tensors) ----
    def forward(self, scene: Scene, camera: Camera, options: Optional[RenderOptions] = None, image=None,
                radii=None, want_stats: bool = False):
        import torch

        if image is None:
            image = torch.empty((camera.height, camera.width, 3), dtype=torch.float32, device=scene.means.device)
        st = _lib.fgs_stats() if want_stats else None
        g = self._gaussians(scene)
        cam = _camera_struct(camera)
        o = _render_options(options, getattr(scene, "background", None))
        rc = self._L.fgs_forward(self._h, C.byref(g), C.byref(cam), C.byref(o), C.c_void_p(_ptr(image)),
                                 C.c_void_p(_ptr(radii)), C.byref(st) if st is not None else None)
        self._check(rc)
        return image, (_stats(st) if st is not None else None)

    def backward(self, scene: Scene, camera: Camera, dl_dimage, options: Optional[BackwardOptions] = None,
                 grads=None, accumulate: bool = False):
        """Returns the flat field-major gradient buffer (59*N floats; see ``split_grads``)."""
        import torch

        n = scene.n
        if tuple(dl_dimage.shape) != (camera.height, camera.width, 3):
            raise InvalidArgument("rasterize_backward: image gradient shape does not match context")
        if grads is None:
            grads = torch.zeros(59 * n, dtype=torch.float32, device=scene.means.device)
        gs = _grad_struct(grads, n)
        cam = _camera_struct(camera)
        o = _backward_options(options, accumulate)
        rc = self._L.fgs_backward(self._h, C.byref(self._gaussians(scene)), C.byref(cam),
                                  C.c_void_p(_ptr(dl_dimage)), C.byref(o), C.byref(gs))
        self._check(rc)
        return grads

    def fwd_bwd_views(self, scene: Scene, cameras, dl_dimages, render_options: Optional[RenderOptions] = None,
                      backward_options: Optional[BackwardOptions] = None, grads=None, comm=None, images=None,
                      accumulate: bool = False):
        """This rank's multi-view step through the C ABI (fgs_fwd_bwd_views): forward + backward of
        every camera, the gradients accumulated into one 59*N buffer and, with a ``Communicator``,
        summed over the ranks by NCCL (the last view's gradient ranges all-reduced while the next
        range is computed). Returns the gradient buffer."""
        import torch

        n = scene.n
        if grads is None:
            grads = torch.zeros(59 * n, dtype=torch.float32, device=scene.means.device)
        nv = len(cameras)
        cams = (_lib.fgs_camera * max(nv, 1))(*[_camera_struct(c) for c in cameras])
        for c, d in zip(cameras, dl_dimages):
            if tuple(d.shape) != (c.height, c.width, 3):
                raise InvalidArgument("rasterize_backward: image gradient shape does not match context")
        dls = (C.c_void_p * max(nv, 1))(*[_ptr(d) for d in dl_dimages])
        imgs = (C.c_void_p * max(nv, 1))(*[(_ptr(images[i]) if images is not None else None) for i in range(nv)])
        ro = _render_options(render_options, getattr(scene, "background", None))
        bo = _backward_options(backward_options, accumulate)
        gs = _grad_struct(grads, n)
        rc = self._L.fgs_fwd_bwd_views(self._h, comm._h if comm is not None else None, C.byref(self._gaussians(scene)),
                                       cams, nv, dls, C.byref(ro), C.byref(bo), C.byref(gs),
                                       imgs if images is not None else None)
        self._check(rc)
        return grads

    # ---- host path (numpy), the reference's calling convention ----
    def render_host(self, scene: Scene, camera: Camera, options: Optional[RenderOptions] = None, radii=True,
                    image=None, want_stats=True):
        s = scene.astype(np.float32)
        if image is None:
            image = np.empty((camera.height, camera.width, 3), np.float32)
        r = np.empty(s.n, np.int32) if radii is True else radii
        st = _lib.fgs_stats() if want_stats else None
        g = self._gaussians(s)
        cam = _camera_struct(camera)
        o = _render_options(options, s.background)
        rc = self._L.fgs_render_host(self._h, C.byref(g), C.byref(cam), C.byref(o), C.c_void_p(_ptr(image)),
                                     C.c_void_p(_ptr(r)), C.byref(st) if st is not None else None)
        self._check(rc)
        return image, r, (_stats(st) if st is not None else None)

    def render_host_async(self, scene: Scene, camera: Camera, options: Optional[RenderOptions] = None, radii=None,
                          image=None, want_stats=True):
        """fgs_render_host_async: returns when the frame is queued (statistics known); `image` is
        filled by the time wait() returns. The arrays are kept alive until then."""
        s = scene.astype(np.float32)
        if image is None:
            image = np.empty((camera.height, camera.width, 3), np.float32)
        r = np.empty(s.n, np.int32) if radii is True else radii
        st = _lib.fgs_stats() if want_stats else None
        g = self._gaussians(s)
        cam = _camera_struct(camera)
        o = _render_options(options, s.background)
        rc = self._L.fgs_render_host_async(self._h, C.byref(g), C.byref(cam), C.byref(o), C.c_void_p(_ptr(image)),
                                           C.c_void_p(_ptr(r)), C.byref(st) if st is not None else None)
        self._check(rc)
        self._inflight = getattr(self, "_inflight", [])[-1:] + [(s, image, r)]  # (two frames in flight)
        return image, r, (_stats(st) if st is not None else None)

    def wait(self):
        """fgs_wait: every render_host_async image is in host memory."""
        self._check(self._L.fgs_wait(self._h))
        self._inflight = []

    def backward_host(self, scene: Scene, camera: Camera, dl_dimage, options: Optional[BackwardOptions] = None,
                      grads=None, accumulate=False):
        s = scene.astype(np.float32)
        dl = np.ascontiguousarray(dl_dimage, np.float32)
        if dl.shape != (camera.height, camera.width, 3):
            raise InvalidArgument("rasterize_backward: image gradient shape does not match context")
        if grads is None:
            grads = np.zeros(59 * s.n, np.float32)
        gs = _grad_struct(grads, s.n)
        cam = _camera_struct(camera)
        o = _backward_options(options, accumulate)
        rc = self._L.fgs_backward_host(self._h, C.byref(self._gaussians(s)), C.byref(cam), C.c_void_p(_ptr(dl)),
                                       C.byref(o), C.byref(gs))
        self._check(rc)
        return grads

    def backward_host_async(self, scene: Scene, camera: Camera, dl_dimage, options: Optional[BackwardOptions] = None,
                            grads=None, accumulate=False):
        """fgs_backward_host_async: returns when the backward is queued; `grads` are filled by the
        time wait() returns (the arrays are kept alive until then)."""
        s = scene.astype(np.float32)
        dl = np.ascontiguousarray(dl_dimage, np.float32)
        if dl.shape != (camera.height, camera.width, 3):
            raise InvalidArgument("rasterize_backward: image gradient shape does not match context")
        if grads is None:
            grads = np.zeros(59 * s.n, np.float32)
        gs = _grad_struct(grads, s.n)
        cam = _camera_struct(camera)
        o = _backward_options(options, accumulate)
        rc = self._L.fgs_backward_host_async(self._h, C.byref(self._gaussians(s)), C.byref(cam),
                                             C.c_void_p(_ptr(dl)), C.byref(o), C.byref(gs))
        self._check(rc)
        self._inflight = getattr(self, "_inflight", [])[-3:] + [(s, dl, grads)]
        return grads

    def last_transfer(self) -> dict:
        """PCIe bytes moved by the last render_host / backward_host call (zero copy reads only
        what the kernels touch when the scene arrays are pinned host memory)."""
        out = (C.c_uint64 * 2)()
        self._check(self._L.fgs_last_transfer(self._h, out))
        return {"h2d": int(out[0]), "d2h": int(out[1])}

    # ---- parity / debug exports ----
    def debug(self, name: str, dtype=np.uint32):
        nbytes = self._L.fgs_debug_get(self._h, name.encode(), None, 0)
        if nbytes < 0:
            raise KeyError(name)
        out = np.empty(nbytes // np.dtype(dtype).itemsize, dtype)
        got = self._L.fgs_debug_get(self._h, name.encode(), C.c_void_p(out.ctypes.data), nbytes)
        if got != nbytes:
            raise FgsError(f"debug_get({name}) failed")
        return out

    def timing(self, reset: bool = False) -> dict:
        """Stage times (ms, summed) and kernel launches recorded since the last reset."""
        ms = (C.c_double * 6)()
        calls = (C.c_uint64 * 2)()
        launches = C.c_uint64()
        self._check(self._L.fgs_timing(self._h, ms, calls, C.byref(launches), int(reset)))
        keys = ["preprocess", "binning", "sort", "raster", "raster_backward", "preprocess_backward"]
        return {"ms": dict(zip(keys, list(ms))), "forward_calls": calls[0], "backward_calls": calls[1],
                "launches": launches.value}

    def fp32_peak(self) -> float:
        v = C.c_double()
        self._check(self._L.fgs_measure_fp32_peak(self._h, C.byref(v)))
        return v.value

    def selftest_crmath(self, which: int, begin: int, count: int, seed: int = 0) -> dict:
        """fgs_selftest_crmath: the fast correctly rounded exp (which 0) / atan2 (1, 2) against
        their definition on the device."""
        out = (C.c_uint64 * 3)()
        self._check(self._L.fgs_selftest_crmath(self._h, int(which), int(begin), int(count), int(seed), out))
        return {"checked": out[0], "mismatches": out[1], "slow": out[2]}

    def counts(self) -> dict:
        a = (C.c_int64 * 9)()
        self._check(self._L.fgs_last_counts(self._h, a))
        keys = ["n", "num_splats", "num_intersections", "tiles_x", "tiles_y", "width", "height", "num_culled",
                "num_degenerate"]
        return dict(zip(keys, list(a)))

    def splats(self) -> dict:
        """Per-Gaussian preprocess outputs of the last forward (reference Splat2D fields)."""
        state = self.debug("state_u8", np.uint8).astype(np.int32)
        rec = self.debug("rec", np.float32).reshape(-1, 12)
        r0, r1, r2 = rec[:, 0:4], rec[:, 4:8], rec[:, 8].copy()
        dk = self.debug("depth_key", np.uint32)
        return {
            "state": state,
            "mean_px": r0[:, 0:2].copy(),
            "conic": np.stack([-2.0 * r0[:, 2], r0[:, 3], -2.0 * r1[:, 0]], 1).astype(np.float32),  # record: -a/2, -c/2
            "color": np.stack([r1[:, 2], r1[:, 3], r2], 1),
            "alpha": r1[:, 1].copy(),
            "depth": (dk & np.uint32(0x7FFFFFFF)).view(np.float32),
            "depth_key": dk,
            "radius": self.debug("radius", np.int32),
        }


def _grad_struct(buf, n) -> _lib.fgs_gradients:
    base = _ptr(buf)
    gs = _lib.fgs_gradients()
    off = 0
    for name, k in GRAD_FIELDS:
        setattr(gs, name, base + 4 * off)
        off += k * n
    return gs


def split_grads(buf, n) -> dict:
    """Views of the flat field-major buffer: mean (n,3), rotation (n,4), log_scale (n,3),
    opacity (n,), sh (n,48)."""
    out, off = {}, 0
    for (name, k), key in zip(GRAD_FIELDS, ("mean", "rotation", "log_scale", "opacity", "sh")):
        v = buf[off:off + k * n]
        out[key] = v.reshape(n, k) if k > 1 else v.reshape(n)
        off += k * n
    return out


def grads_as_rows(buf, n) -> np.ndarray:
    """(n, 59) rows in the oracle's order: mean 3, rotation 4, log_scale 3, opacity 1, sh 48."""
    b = np.asarray(buf.cpu().numpy() if hasattr(buf, "cpu") else buf)
    s = split_grads(b, n)
    return np.concatenate([s["mean"], s["rotation"], s["log_scale"], s["opacity"][:, None], s["sh"]], 1)


def _stats(st) -> RenderStats:
    return RenderStats(int(st.num_intersections), int(st.num_splats), int(st.num_culled), int(st.num_degenerate),
                       st.preprocess_ms, st.binning_ms, st.sort_ms, st.raster_ms, int(st.peak_aux_bytes))


@dataclass
class ForwardContext:
    """Everything backward needs (splatting.hpp:309-321): here, the device context itself."""

    rasterizer: Rasterizer
    camera: Camera
    scene_size: int
    sh_degree: int


@dataclass
class RenderResult:
    image: np.ndarray
    stats: RenderStats
    context: ForwardContext
    radii: np.ndarray = field(default=None)


_default: dict = {}


def _default_rasterizer(device=0) -> Rasterizer:
    if device not in _default:
        _default[device] = Rasterizer(device)
    return _default[device]


def render(scene: Scene, camera: Camera, options: Optional[RenderOptions] = None, device: int = 0,
           rasterizer: Optional[Rasterizer] = None) -> RenderResult:
    """render<float> (splatting.hpp:330) on the B200: host arrays in, host image out."""
    r = rasterizer or Rasterizer(device)
    opts = options or RenderOptions()
    image, radii, stats = r.render_host(scene, camera, opts)
    return RenderResult(image, stats, ForwardContext(r, camera, scene.n, opts.sh_degree), radii)


def backward(scene: Scene, camera: Camera, result: RenderResult, dl_dimage,
             options: Optional[BackwardOptions] = None) -> dict:
    """backward<float> (gradients.hpp:207): returns per-Gaussian gradient arrays (host)."""
    ctx = result.context
    if ctx.scene_size != scene.n:
        raise InvalidArgument("backward: forward context was built for a different scene")
    if not ctx.camera.same_as(camera):
        raise InvalidArgument("backward: forward context was built for a different camera")
    buf = ctx.rasterizer.backward_host(scene, camera, dl_dimage, options)
    return split_grads(buf, scene.n)
