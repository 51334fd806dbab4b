"""ctypes binding of the C ABI in include/fgs.h (libfgs.so, built in-tree).

There is no fallback: if the library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfgs.so")
# FGS_LIB=checked selects libfgs_checked.so: the same sources built with -DFGS_CHECKED (device-side
# bounds / invariant checks that trap; tests/test_checked_gpu.py); FGS_LIB=<name>, an experiment
# build libfgs_<name>.so (build.py --variant)
CHECKED_LIB_PATH = os.path.join(HERE, "libfgs_checked.so")

FGS_OK, FGS_EINVAL, FGS_EDEGENERATE_QUAT, FGS_ECUDA, FGS_ENOMEM, FGS_ESTATE, FGS_ENONFINITE = range(7)
FGS_FLAG_COUNTERS, FGS_FLAG_KEEP_KEYS, FGS_FLAG_TIMING, FGS_FLAG_BLEND_COUNT = 1, 2, 4, 8
FGS_FLAG_ROW_SCATTER, FGS_FLAG_SLOT_SCATTER, FGS_FLAG_GLOBAL_SLOTS = 16, 32, 64


class fgs_camera(C.Structure):
    _fields_ = [("model", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float),
                ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float), ("rotation_wc", C.c_float * 9),
                ("translation_wc", C.c_float * 3), ("fov_max", C.c_float)]


class fgs_gaussians(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("rotations", C.c_void_p), ("log_scales", C.c_void_p),
                ("opacity_logits", C.c_void_p), ("sh", C.c_void_p)]


class fgs_gradients(C.Structure):
    _fields_ = [("d_means", C.c_void_p), ("d_rotations", C.c_void_p), ("d_log_scales", C.c_void_p),
                ("d_opacity_logits", C.c_void_p), ("d_sh", C.c_void_p)]


class fgs_render_options(C.Structure):
    _fields_ = [("sh_degree", C.c_int32), ("use_background", C.c_int32), ("background", C.c_float * 3)]


class fgs_backward_options(C.Structure):
    _fields_ = [("jacobian_grad_scale", C.c_float * 3), ("full_sh", C.c_int32), ("accumulate", C.c_int32),
                ("sh_view_dir_grad", C.c_int32)]


class fgs_stats(C.Structure):
    _fields_ = [("num_intersections", C.c_uint64), ("num_splats", C.c_uint32), ("num_culled", C.c_uint32),
                ("num_degenerate", C.c_uint32), ("preprocess_ms", C.c_double), ("binning_ms", C.c_double),
                ("sort_ms", C.c_double), ("raster_ms", C.c_double), ("peak_aux_bytes", C.c_uint64)]


class fgs_params(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("rotations", C.c_void_p), ("log_scales", C.c_void_p),
                ("opacity_logits", C.c_void_p), ("sh", C.c_void_p)]


class fgs_adam_options(C.Structure):
    _fields_ = [(k, C.c_float) for k in ("lr_mean", "lr_rotation", "lr_log_scale", "lr_opacity", "lr_sh_dc",
                                         "lr_sh_rest", "beta1", "beta2", "eps")]


class fgs_adam_state(C.Structure):
    _fields_ = [("step", C.c_int64), ("m", fgs_gradients), ("v", fgs_gradients)]


class fgs_gaussians_aos(C.Structure):
    _fields_ = [("n", C.c_int64), ("data", C.c_void_p), ("stride", C.c_int64), ("off_mean", C.c_int64),
                ("off_rotation", C.c_int64), ("off_log_scale", C.c_int64), ("off_opacity_logit", C.c_int64),
                ("off_sh", C.c_int64)]


class fgs_train_options(C.Structure):
    _fields_ = [("sh_degree", C.c_int32), ("background", C.c_float * 3), ("lam", C.c_float),
                ("adam", fgs_adam_options)]


EXPORTS = ["fgs_create", "fgs_destroy", "fgs_set_stream", "fgs_last_error", "fgs_forward", "fgs_backward",
           "fgs_render_host", "fgs_backward_host", "fgs_set_flags", "fgs_debug_get", "fgs_last_counts",
           "fgs_timing", "fgs_measure_fp32_peak", "fgs_l1_dssim_loss", "fgs_adam_step", "fgs_train_step",
           "fgs_bruteforce_render", "fgs_bruteforce_render_f64", "fgs_last_transfer", "fgs_render_host_aos",
           "fgs_backward_host_aos", "fgs_comm_get_unique_id", "fgs_comm_init", "fgs_comm_init_all",
           "fgs_comm_destroy", "fgs_allreduce_gradients", "fgs_fwd_bwd_views", "fgs_selftest_crmath",
           "fgs_render_host_async", "fgs_backward_host_async", "fgs_wait"]

_lib = None


def load(path: str | None = None):
    """Load libfgs.so (libfgs_checked.so with FGS_LIB=checked) and declare its signatures. Raises
    if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if path is None:
        v = os.environ.get("FGS_LIB")
        path = os.path.join(HERE, f"libfgs_{v}.so") if v else LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -m paper_2409_04751_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, i32 = C.c_void_p, C.c_int
    P = C.POINTER
    L.fgs_create.argtypes = [i32, P(vp)]
    L.fgs_create.restype = i32
    L.fgs_destroy.argtypes = [vp]
    L.fgs_destroy.restype = i32
    L.fgs_set_stream.argtypes = [vp, vp]
    L.fgs_set_stream.restype = i32
    L.fgs_set_flags.argtypes = [vp, C.c_uint32]
    L.fgs_set_flags.restype = i32
    L.fgs_last_error.argtypes = [vp]
    L.fgs_last_error.restype = C.c_char_p
    fwd = [vp, P(fgs_gaussians), P(fgs_camera), P(fgs_render_options), vp, vp, P(fgs_stats)]
    bwd = [vp, P(fgs_gaussians), P(fgs_camera), vp, P(fgs_backward_options), P(fgs_gradients)]
    for name, args in (("fgs_forward", fwd), ("fgs_render_host", fwd), ("fgs_render_host_async", fwd),
                       ("fgs_backward", bwd), ("fgs_backward_host", bwd), ("fgs_backward_host_async", bwd)):
        getattr(L, name).argtypes = args
        getattr(L, name).restype = i32
    L.fgs_debug_get.argtypes = [vp, C.c_char_p, vp, C.c_int64]
    L.fgs_debug_get.restype = C.c_int64
    L.fgs_last_counts.argtypes = [vp, P(C.c_int64)]
    L.fgs_last_counts.restype = i32
    L.fgs_timing.argtypes = [vp, P(C.c_double), P(C.c_uint64), P(C.c_uint64), i32]
    L.fgs_timing.restype = i32
    L.fgs_measure_fp32_peak.argtypes = [vp, P(C.c_double)]
    L.fgs_wait.argtypes = [vp]
    L.fgs_wait.restype = i32
    L.fgs_selftest_crmath.argtypes = [vp, i32, C.c_uint64, C.c_uint64, C.c_uint64, P(C.c_uint64)]
    L.fgs_selftest_crmath.restype = i32
    L.fgs_measure_fp32_peak.restype = i32
    L.fgs_l1_dssim_loss.argtypes = [vp, vp, vp, C.c_int32, C.c_int32, C.c_float, vp, P(C.c_double)]
    L.fgs_l1_dssim_loss.restype = i32
    L.fgs_adam_step.argtypes = [vp, P(fgs_params), P(fgs_gradients), P(fgs_adam_state), P(fgs_adam_options)]
    L.fgs_adam_step.restype = i32
    L.fgs_train_step.argtypes = [vp, P(fgs_params), P(fgs_camera), vp, P(fgs_train_options), P(fgs_adam_state),
                                 P(C.c_double)]
    L.fgs_train_step.restype = i32
    L.fgs_bruteforce_render.argtypes = [vp, P(fgs_gaussians), P(fgs_camera), C.c_int32, P(C.c_double), vp, vp]
    L.fgs_bruteforce_render.restype = i32
    L.fgs_bruteforce_render_f64.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, P(fgs_camera), C.c_int32,
                                            P(C.c_double), vp, vp]
    L.fgs_bruteforce_render_f64.restype = i32
    L.fgs_render_host_aos.argtypes = [vp, P(fgs_gaussians_aos), P(fgs_camera), P(fgs_render_options), vp, vp,
                                      P(fgs_stats)]
    L.fgs_render_host_aos.restype = i32
    L.fgs_backward_host_aos.argtypes = [vp, P(fgs_gaussians_aos), P(fgs_camera), vp, P(fgs_backward_options),
                                        P(fgs_gradients)]
    L.fgs_backward_host_aos.restype = i32
    L.fgs_comm_get_unique_id.argtypes = [P(C.c_uint8)]
    L.fgs_comm_get_unique_id.restype = i32
    L.fgs_comm_init.argtypes = [vp, P(C.c_uint8), i32, i32, P(vp)]
    L.fgs_comm_init.restype = i32
    L.fgs_comm_init_all.argtypes = [P(vp), i32, P(vp)]
    L.fgs_comm_init_all.restype = i32
    L.fgs_comm_destroy.argtypes = [vp]
    L.fgs_comm_destroy.restype = i32
    L.fgs_allreduce_gradients.argtypes = [vp, P(fgs_gradients), C.c_int64]
    L.fgs_allreduce_gradients.restype = i32
    L.fgs_fwd_bwd_views.argtypes = [vp, vp, P(fgs_gaussians), P(fgs_camera), i32, P(vp), P(fgs_render_options),
                                    P(fgs_backward_options), P(fgs_gradients), P(vp)]
    L.fgs_fwd_bwd_views.restype = i32
    L.fgs_last_transfer.argtypes = [vp, P(C.c_uint64)]
    L.fgs_last_transfer.restype = i32
    _lib = L
    return L
