"""ctypes loader for the CPU oracle (oracle/fgs_oracle.cpp) and the reference build.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline leg, never by the product package.

Two libraries:
  * ``oracle/_build/libfgs_oracle.so`` — the restatement (parity / libm modes).
  * ``oracle/_ref/libomnisplat_ref.so`` — the reference's own headers compiled against the
    repo's Eigen-subset shim (built here by oracle/Makefile when /root/reference exists; the
    built .so travels to the GPU box). ``ref_available()`` says whether it is present.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libfgs_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libomnisplat_ref.so")

MODE_PARITY = 0
MODE_LIBM = 1

_lib = None
_ref = None


def build(quiet=True):
    """Build the oracle (and, when /root/reference is mounted, the reference) via make."""
    # make's messages go to stderr: callers such as bench.py print one JSON line on stdout
    subprocess.run(["make", "-C", HERE] + (["-s"] if quiet else []), check=True, stdout=sys.stderr)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, dp, fp = C.c_void_p, C.c_int64, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_float)
        for name, rp in (("orc_render_f32", fp), ("orc_render_f64", dp)):
            fn = getattr(L, name)
            fn.restype = vp
            fn.argtypes = [i64, rp, rp, rp, rp, rp, dp, rp, i32, i32, i32]
        for name, rp in (("orc_backward_f32", fp), ("orc_backward_f64", dp)):
            fn = getattr(L, name)
            fn.restype = i32
            fn.argtypes = [vp, i64, rp, rp, dp, i32, i32, i32, i32, rp]
        L.orc_free.argtypes = [vp]
        L.orc_sizes.argtypes = [vp, C.POINTER(C.c_int64)]
        L.orc_stats.argtypes = [vp, dp]
        L.orc_get.restype = i64
        L.orc_get.argtypes = [vp, C.c_char_p, vp]
        L.orc_last_error.restype = C.c_char_p
        L.orc_bruteforce_render_f64.restype = i32
        L.orc_bruteforce_render_f64.argtypes = [i64, dp, dp, dp, dp, dp, dp, dp, i32, dp, dp]
        L.orc_bruteforce_intersections.restype = C.c_uint64
        L.orc_bruteforce_intersections.argtypes = [i64, dp, C.POINTER(C.c_int32), i32, i32]
        L.orc_project_f64.restype = i32
        L.orc_project_f64.argtypes = [dp, dp, dp, dp, i32]
        L.orc_project_f32.restype = i32
        L.orc_project_f32.argtypes = [dp, fp, fp, fp, i32]
        L.orc_jacobian_grad_f64.argtypes = [dp, dp, dp]
        L.orc_build_covariance_f64.restype = i32
        L.orc_build_covariance_f64.argtypes = [dp, dp, dp]
        L.orc_build_covariance_backward_f64.restype = i32
        L.orc_build_covariance_backward_f64.argtypes = [dp, dp, dp, dp, dp]
        L.orc_eval_sh_f64.argtypes = [dp, dp, i32, dp]
        L.orc_splats_render_f64.restype = vp
        L.orc_splats_render_f64.argtypes = [i64, dp, dp, dp, C.POINTER(C.c_int32), dp, dp, i32, i32, dp, i32]
        L.orc_splats_backward_f64.restype = i32
        L.orc_splats_backward_f64.argtypes = [vp, dp, dp, i32]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref_lib():
    """The reference headers compiled against the Eigen shim (same C entry points as the
    restatement's render/backward/get/stats, prefixed ``ref_``)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(REF_PATH)
        L = C.CDLL(REF_PATH)
        vp, i64, i32, dp, fp = C.c_void_p, C.c_int64, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_float)
        for name, rp in (("ref_render_f32", fp), ("ref_render_f64", dp)):
            fn = getattr(L, name)
            fn.restype = vp
            fn.argtypes = [i64, rp, rp, rp, rp, rp, dp, rp, i32, i32]
        for name, rp in (("ref_backward_f32", fp), ("ref_backward_f64", dp)):
            fn = getattr(L, name)
            fn.restype = i32
            fn.argtypes = [vp, i64, rp, rp, dp, i32, rp]
        L.ref_free.argtypes = [vp]
        L.ref_sizes.argtypes = [vp, C.POINTER(C.c_int64)]
        L.ref_stats.argtypes = [vp, dp]
        L.ref_get.restype = i64
        L.ref_get.argtypes = [vp, C.c_char_p, vp]
        L.ref_last_error.restype = C.c_char_p
        L.ref_bruteforce_render_f64.restype = i32
        L.ref_bruteforce_render_f64.argtypes = [i64, dp, dp, dp, dp, dp, dp, dp, i32, dp]
        _ref = L
    return _ref


class OracleError(RuntimeError):
    pass


_DTYPES = {
    "state": np.int32, "radius": np.int32, "source": np.int32,
    "refs": np.uint32, "offsets": np.uint32, "key_tile": np.uint32, "key_splat": np.uint32,
    "key_depth": np.uint64, "count": np.uint16,
}


@dataclass
class Result:
    """A forward render held by the oracle (ForwardContext analogue)."""

    handle: int
    dtype: type
    n: int
    num_splats: int
    num_intersections: int
    tiles_x: int
    tiles_y: int
    width: int
    height: int
    prefix: str = "orc"

    def _L(self):
        return lib() if self.prefix == "orc" else ref_lib()

    def get(self, name):
        L = self._L()
        fn = L.orc_get if self.prefix == "orc" else L.ref_get
        cnt = fn(self.handle, name.encode(), None)
        if cnt < 0:
            raise KeyError(name)
        out = np.empty(cnt, _DTYPES.get(name, self.dtype))
        fn(self.handle, name.encode(), out.ctypes.data_as(C.c_void_p))
        return out

    def stats(self) -> dict:
        out = np.zeros(11, np.float64)
        (self._L().orc_stats if self.prefix == "orc" else self._L().ref_stats)(self.handle, _p(out, C.c_double))
        keys = ["num_intersections", "num_splats", "num_culled", "num_degenerate", "preprocess_ms",
                "binning_ms", "sort_ms", "raster_ms", "peak_aux_bytes", "e_eval", "e_contrib"]
        return dict(zip(keys, out.tolist()))

    @property
    def image(self):
        return self.get("image").reshape(self.height, self.width, 3)

    def close(self):
        if self.handle:
            (self._L().orc_free if self.prefix == "orc" else self._L().ref_free)(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _scene_arrays(scene, dtype):
    s = scene.astype(dtype)
    return s, [s.means, s.rotations, s.log_scales, s.opacity_logits, s.sh]


def render(scene, camera, sh_degree=3, background=None, dtype=np.float32, threads=0, mode=MODE_PARITY,
           impl="orc") -> Result:
    """Reference ``render<S>`` (inc/splatting.hpp:330-374) on the oracle (``impl='orc'``) or on
    the reference build (``impl='ref'``; always libm transcendentals)."""
    ct = C.c_float if dtype == np.float32 else C.c_double
    s, arrs = _scene_arrays(scene, dtype)
    bg = np.asarray(s.background if background is None else background, dtype)
    cam = camera.to_array()
    if impl == "orc":
        L = lib()
        fn = L.orc_render_f32 if dtype == np.float32 else L.orc_render_f64
        h = fn(s.n, *[_p(a, ct) for a in arrs], _p(cam, C.c_double), _p(bg, ct), sh_degree, threads, mode)
        err = L.orc_last_error
        sizes_fn = L.orc_sizes
    else:
        L = ref_lib()
        fn = L.ref_render_f32 if dtype == np.float32 else L.ref_render_f64
        h = fn(s.n, *[_p(a, ct) for a in arrs], _p(cam, C.c_double), _p(bg, ct), sh_degree, threads)
        err = L.ref_last_error
        sizes_fn = L.ref_sizes
    if not h:
        raise OracleError(err().decode())
    sz = np.zeros(7, np.int64)
    sizes_fn(h, sz.ctypes.data_as(C.POINTER(C.c_int64)))
    return Result(h, dtype, int(sz[0]), int(sz[1]), int(sz[2]), int(sz[3]), int(sz[4]), int(sz[5]),
                  int(sz[6]), impl)


def backward(res: Result, n, dl_dimage, full_sh=True, jacobian_grad_scale=None, threads=0,
             mode=MODE_PARITY, want_splat_grads=False, sh_view_dir_grad=False):
    """Reference ``backward<S>`` (inc/gradients.hpp:207-267). Returns (grads[n,59], splat_grads
    [num_splats,9] or None)."""
    dtype = res.dtype
    ct = C.c_float if dtype == np.float32 else C.c_double
    dl = np.ascontiguousarray(dl_dimage, dtype).reshape(-1)
    grads = np.zeros((n, 59), dtype)
    sg = np.zeros((res.num_splats, 9), dtype) if want_splat_grads else None
    jgs = None if jacobian_grad_scale is None else np.asarray(jacobian_grad_scale, np.float64)
    jp = _p(jgs, C.c_double) if jgs is not None else None
    if res.prefix == "orc":
        L = lib()
        fn = L.orc_backward_f32 if dtype == np.float32 else L.orc_backward_f64
        rc = fn(res.handle, n, _p(dl, ct), _p(grads, ct), jp, int(full_sh), int(sh_view_dir_grad), threads, mode,
                _p(sg, ct) if sg is not None else None)
        err = L.orc_last_error
    else:
        L = ref_lib()
        fn = L.ref_backward_f32 if dtype == np.float32 else L.ref_backward_f64
        rc = fn(res.handle, n, _p(dl, ct), _p(grads, ct), jp, threads, _p(sg, ct) if sg is not None else None)
        err = L.ref_last_error
    if rc != 0:
        raise OracleError(err().decode())
    return grads, sg


def bruteforce_render(scene, camera, sh_degree=0, background=None, impl="orc"):
    """inc/oracle.hpp:231-270 in double. Returns (image[H,W,3], transmittance[H,W])."""
    s, arrs = _scene_arrays(scene, np.float64)
    bg = np.asarray(s.background if background is None else background, np.float64)
    cam = camera.to_array()
    img = np.zeros((camera.height, camera.width, 3))
    tr = np.zeros((camera.height, camera.width))
    dp = C.c_double
    if impl == "orc":
        L = lib()
        rc = L.orc_bruteforce_render_f64(s.n, *[_p(a, dp) for a in arrs], _p(cam, dp), _p(bg, dp), sh_degree,
                                         _p(img, dp), _p(tr, dp))
        err = L.orc_last_error
    else:
        L = ref_lib()
        rc = L.ref_bruteforce_render_f64(s.n, *[_p(a, dp) for a in arrs], _p(cam, dp), _p(bg, dp), sh_degree,
                                         _p(img, dp))
        err = L.ref_last_error
    if rc != 0:
        raise OracleError(err().decode())
    return img, tr


def bruteforce_intersections(mean_px, radius, width, height) -> int:
    m = np.ascontiguousarray(mean_px, np.float64).reshape(-1)
    r = np.ascontiguousarray(radius, np.int32)
    return int(lib().orc_bruteforce_intersections(len(r), _p(m, C.c_double), _p(r, C.c_int32), width, height))


def project(camera, p, force=0):
    """cameras.hpp:139-177 in double: (visible, pixel[2], jacobian[2,3])."""
    cam = camera.to_array()
    pt = np.ascontiguousarray(p, np.float64)
    px = np.zeros(2)
    j = np.zeros((2, 3))
    v = lib().orc_project_f64(_p(cam, C.c_double), _p(pt, C.c_double), _p(px, C.c_double), _p(j, C.c_double), force)
    return bool(v), px, j


def jacobian_grad(camera, p):
    cam = camera.to_array()
    pt = np.ascontiguousarray(p, np.float64)
    out = np.zeros((3, 2, 3))
    lib().orc_jacobian_grad_f64(_p(cam, C.c_double), _p(pt, C.c_double), _p(out, C.c_double))
    return out


def build_covariance(q, s):
    q = np.ascontiguousarray(q, np.float64)
    s = np.ascontiguousarray(s, np.float64)
    out = np.zeros((3, 3))
    if lib().orc_build_covariance_f64(_p(q, C.c_double), _p(s, C.c_double), _p(out, C.c_double)) != 0:
        raise ValueError(lib().orc_last_error().decode())
    return out


def build_covariance_backward(q, s, g):
    q = np.ascontiguousarray(q, np.float64)
    s = np.ascontiguousarray(s, np.float64)
    g = np.ascontiguousarray(g, np.float64)
    dq = np.zeros(4)
    ds = np.zeros(3)
    if lib().orc_build_covariance_backward_f64(_p(q, C.c_double), _p(s, C.c_double), _p(g, C.c_double),
                                               _p(dq, C.c_double), _p(ds, C.c_double)) != 0:
        raise ValueError(lib().orc_last_error().decode())
    return dq, ds


def eval_sh(sh48, d, degree):
    sh = np.ascontiguousarray(sh48, np.float64)
    dd = np.ascontiguousarray(d, np.float64)
    out = np.zeros(3)
    lib().orc_eval_sh_f64(_p(sh, C.c_double), _p(dd, C.c_double), degree, _p(out, C.c_double))
    return out


def splats_render(mean_px, conic, depth, radius, color, alpha, width, height, background=(0, 0, 0), threads=0):
    """bin_and_sort + rasterize (inc/splatting.hpp:196-306) over explicit splats, in double."""
    f = lambda a, k: np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, k) if k > 1 else np.asarray(a, np.float64).reshape(-1))
    m, c, d, col, al = f(mean_px, 2), f(conic, 3), f(depth, 1), f(color, 3), f(alpha, 1)
    r = np.ascontiguousarray(radius, np.int32).reshape(-1)
    bg = np.asarray(background, np.float64)
    dp = C.c_double
    L = lib()
    h = L.orc_splats_render_f64(len(r), _p(m, dp), _p(c, dp), _p(d, dp), _p(r, C.c_int32), _p(col, dp), _p(al, dp),
                                width, height, _p(bg, dp), threads)
    sz = np.zeros(7, np.int64)
    L.orc_sizes(h, sz.ctypes.data_as(C.POINTER(C.c_int64)))
    return Result(h, np.float64, int(sz[0]), int(sz[1]), int(sz[2]), int(sz[3]), int(sz[4]), int(sz[5]), int(sz[6]))


def splats_backward(res: Result, dl_dimage, threads=0):
    """rasterize_backward (inc/gradients.hpp:69-175) -> (num_splats, 9) splat gradients."""
    dl = np.ascontiguousarray(dl_dimage, np.float64).reshape(-1)
    out = np.zeros((res.num_splats, 9))
    if lib().orc_splats_backward_f64(res.handle, _p(dl, C.c_double), _p(out, C.c_double), threads) != 0:
        raise OracleError(lib().orc_last_error().decode())
    return out


# ---------------------------------------------------------------------------------------
# Training-step oracle: numpy restatements of the reference's loss and
# optimizer, and wrappers around the reference's own code (oracle/_ref) that pin them.

SSIM_WINDOW, SSIM_SIGMA, SSIM_C1, SSIM_C2 = 11, 1.5, 0.01 ** 2, 0.03 ** 2  # inc/metrics.hpp:18-21


def _ssim_window():
    """inc/metrics.hpp:23-34: normalised 11-tap Gaussian, sigma 1.5."""
    d = np.arange(SSIM_WINDOW, dtype=np.float64) - SSIM_WINDOW // 2
    w = np.exp(-d * d / (2.0 * SSIM_SIGMA * SSIM_SIGMA))
    return w / w.sum()


def _blur(plane):
    """inc/metrics.hpp:37-61: separable zero-padded filter (rows, then columns)."""
    w = _ssim_window()
    r = SSIM_WINDOW // 2
    h, wd = plane.shape
    pad = np.zeros((h, wd + 2 * r))
    pad[:, r:r + wd] = plane
    tmp = sum(w[k] * pad[:, k:k + wd] for k in range(SSIM_WINDOW))
    pad = np.zeros((h + 2 * r, wd))
    pad[r:r + h, :] = tmp
    return sum(w[k] * pad[k:k + h, :] for k in range(SSIM_WINDOW))


def ssim(rendered, target, want_grad=False):
    """inc/metrics.hpp:86-161: mean SSIM over the 11x11 Gaussian-window map per channel,
    averaged; optionally d(mean SSIM)/d(rendered) in the difference-factored form."""
    x_img = np.asarray(rendered, np.float64)
    y_img = np.asarray(target, np.float64)
    h, w, _ = x_img.shape
    norm = 1.0 / (h * w * 3)
    total = 0.0
    grad = np.zeros_like(x_img) if want_grad else None
    for ch in range(3):
        x, y = x_img[:, :, ch], y_img[:, :, ch]
        mx, my = _blur(x), _blur(y)
        mxx, myy, mxy = _blur(x * x), _blur(y * y), _blur(x * y)
        sx2, sy2, sxy = mxx - mx * mx, myy - my * my, mxy - mx * my
        n1 = 2 * mx * my + SSIM_C1
        n2 = 2 * sxy + SSIM_C2
        d1 = mx * mx + my * my + SSIM_C1
        d2 = sx2 + sy2 + SSIM_C2
        s = (n1 * n2) / (d1 * d2)
        total += s.sum()
        if want_grad:
            a = 2 * n2 * (my - mx) * (my * (mx + my) + SSIM_C1) / (d1 * d1 * d2)
            b = -s / d2
            e = 2 * n1 * (d2 - n2) / (d1 * d2 * d2)
            ca, cb, cbdmu, ce, cemy = _blur(a), _blur(b), _blur(b * (mx - my)), _blur(e), _blur(e * my)
            grad[:, :, ch] = norm * (ca + 2 * (x - y) * cb - 2 * cbdmu + y * ce - cemy)
    return total * norm, grad


def l1_dssim_loss(rendered, target, lam=0.2):
    """inc/metrics.hpp:172-195: L = (1 - lam) L1 + lam (1 - SSIM) and dL/drendered.
    Returns (total, l1, dssim, d_rendered)."""
    x = np.asarray(rendered, np.float64)
    y = np.asarray(target, np.float64)
    norm = 1.0 / x.size
    s, ds = ssim(x, y, want_grad=True)
    diff = x - y
    l1 = np.abs(diff).sum() * norm
    d = (1.0 - lam) * np.sign(diff) * norm - lam * ds
    return (1.0 - lam) * l1 + lam * (1.0 - s), l1, 1.0 - s, d


ADAM_BETA1, ADAM_BETA2, ADAM_EPS = 0.9, 0.999, 1e-15  # inc/optimize.hpp:72-76
PARAM_GROUPS = {"mean": slice(0, 3), "rotation": slice(3, 7), "log_scale": slice(7, 10), "opacity": slice(10, 11),
                "sh_dc": [11, 27, 43], "sh_rest": [c * 16 + j + 11 for c in range(3) for j in range(1, 16)]}


def adam_step(params, grads, m, v, step, lr):
    """inc/optimize.hpp:100-145 on (N, 59) rows in place; lr maps PARAM_GROUPS names to rates
    (the reference has no sh_rest group: rate 0 / absent leaves those rows untouched).
    ``step`` is the state's step before the call; returns the new step."""
    step += 1
    bc1 = 1.0 - ADAM_BETA1 ** step
    bc2 = 1.0 - ADAM_BETA2 ** step
    for name, sl in PARAM_GROUPS.items():
        rate = lr.get(name, 0.0)
        if not rate:
            continue
        g = grads[:, sl]
        m[:, sl] = ADAM_BETA1 * m[:, sl] + (1 - ADAM_BETA1) * g
        v[:, sl] = ADAM_BETA2 * v[:, sl] + (1 - ADAM_BETA2) * g * g
        params[:, sl] -= rate * (m[:, sl] / bc1) / (np.sqrt(v[:, sl] / bc2) + ADAM_EPS)
    return step


def ref_l1_dssim_loss(rendered, target, lam=0.2):
    """The reference's own l1_dssim_loss (inc/metrics.hpp:172-195) via oracle/_ref."""
    L = ref_lib()
    x = np.ascontiguousarray(rendered, np.float64)
    y = np.ascontiguousarray(target, np.float64)
    h, w, _ = x.shape
    d = np.zeros_like(x)
    out = np.zeros(3)
    dp = C.POINTER(C.c_double)
    fn = L.ref_l1_dssim_loss_f64
    fn.restype = C.c_int
    fn.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, dp, dp]
    if fn(w, h, _p(x, C.c_double), _p(y, C.c_double), lam, _p(d, C.c_double), _p(out, C.c_double)) != 0:
        raise OracleError(L.ref_last_error().decode())
    return out[0], out[1], out[2], d


def ref_adam_step(params, grads, m, v, step, lr):
    """The reference's own adam_step (inc/optimize.hpp:115-145) via oracle/_ref, in place on
    (N, 59) float64 rows (mean, rotation, log_scale, opacity, sh_dc updated)."""
    L = ref_lib()
    fn = L.ref_adam_step_f64
    dp = C.POINTER(C.c_double)
    fn.restype = C.c_int
    fn.argtypes = [C.c_int64, dp, dp, dp, dp, C.c_int64, dp]
    rates = np.array([lr["mean"], lr["rotation"], lr["log_scale"], lr["opacity"], lr["sh_dc"]], np.float64)
    for a in (params, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = np.ascontiguousarray(grads, np.float64)
    if fn(params.shape[0], _p(params, C.c_double), _p(g, C.c_double), _p(m, C.c_double), _p(v, C.c_double), step,
          _p(rates, C.c_double)) != 0:
        raise OracleError(L.ref_last_error().decode())
    return step + 1
