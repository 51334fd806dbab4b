"""Python mirror of the host I/O in include/fgs_io.hpp: the reference's scene PLY and camera
JSON formats.

  load_ply / save_ply          src/ply_io.cpp:40-145  (3DGS binary_little_endian layout)
  load_cameras / save_cameras  src/camera_io.cpp:25-127

Errors are RuntimeError with the reference's messages; warnings are returned, as the
reference's PlyReadResult / CameraReadResult do.
"""
from __future__ import annotations

import json
import math

import numpy as np

from .types import CAMERA_FISHEYE, CAMERA_PANORAMA, CAMERA_PINHOLE, Camera, Scene

FULL_PROPS = (["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"] +
              [f"f_rest_{i}" for i in range(45)] +
              ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"])
DC_PROPS = ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1",
            "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
MODEL_NAMES = {CAMERA_PINHOLE: "pinhole", CAMERA_FISHEYE: "fisheye_equidistant", CAMERA_PANORAMA: "panorama"}


def _sh_to_ply_rest(sh):
    """(N,48) [channel*16 + basis] -> f_rest order c*15 + (j-1) (src/ply_io.cpp:109-117)."""
    sh = sh.reshape(-1, 3, 16)
    return sh[:, :, 1:].reshape(-1, 45)


def save_ply(scene: Scene, path: str) -> None:
    n = scene.n
    rows = np.zeros((n, 62), np.float32)
    rows[:, 0:3] = scene.means
    sh = np.asarray(scene.sh, np.float32).reshape(n, 3, 16)
    rows[:, 6:9] = sh[:, :, 0]
    rows[:, 9:54] = _sh_to_ply_rest(sh)
    rows[:, 54] = scene.opacity_logits
    rows[:, 55:58] = scene.log_scales
    rows[:, 58:62] = scene.rotations
    with open(path, "wb") as f:
        f.write(f"ply\nformat binary_little_endian 1.0\nelement vertex {n}\n".encode())
        for p in FULL_PROPS:
            f.write(f"property float {p}\n".encode())
        f.write(b"end_header\n")
        f.write(rows.astype("<f4").tobytes())


def load_ply(path: str):
    """Returns (Scene, warnings)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"load_ply: cannot open {path}")
    with f:
        first = f.readline().decode("latin1").rstrip("\n")
        if first not in ("ply", "ply\r"):
            raise RuntimeError(f"load_ply: {path} is not a PLY file")
        count, fmt_seen, props = 0, False, []
        while True:
            raw = f.readline()
            if not raw:
                break
            line = raw.decode("latin1").rstrip("\n").rstrip("\r")
            if line == "end_header":
                break
            words = line.split()
            word = words[0] if words else ""
            if word == "format":
                fmt = words[1] if len(words) > 1 else ""
                if fmt != "binary_little_endian":
                    raise RuntimeError(f"load_ply: binary_little_endian required, got format '{fmt}'")
                fmt_seen = True
            elif word == "element":
                if words[1] != "vertex":
                    raise RuntimeError(f"load_ply: unsupported element '{words[1]}'")
                count = int(words[2])
            elif word == "property":
                if words[1] != "float":
                    raise RuntimeError(f"load_ply: property '{words[2]}' has type '{words[1]}', expected float")
                props.append(words[2])
            elif word in ("comment", "obj_info", ""):
                continue
            else:
                raise RuntimeError(f"load_ply: unexpected header line '{line}'")
        if not fmt_seen:
            raise RuntimeError("load_ply: missing format line (binary_little_endian required)")
        warnings = []
        if props == FULL_PROPS:
            has_rest = True
        elif props == DC_PROPS:
            has_rest = False
            warnings.append("load_ply: f_rest_* properties missing; higher-order SH set to zero")
        else:
            raise RuntimeError("load_ply: unknown property layout; expected [" + ",".join(FULL_PROPS) +
                               "] (or the f_rest-free variant), found [" + ",".join(props) + "]")
        start = f.tell()
        stride = len(props)
        data = f.read(count * stride * 4)
    if len(data) != count * stride * 4:
        full = len(data) // (stride * 4)
        raise RuntimeError(f"load_ply: truncated payload at byte offset {start + len(data)}"
                           if full < count else "load_ply: truncated payload")
    rows = np.frombuffer(data, "<f4").reshape(count, stride).astype(np.float32)
    sh = np.zeros((count, 3, 16), np.float32)
    sh[:, :, 0] = rows[:, 6:9]
    k = 9
    if has_rest:
        sh[:, :, 1:] = rows[:, 9:54].reshape(count, 3, 15)
        k = 54
    scene = Scene(np.ascontiguousarray(rows[:, 0:3]), np.ascontiguousarray(rows[:, k + 4:k + 8]),
                  np.ascontiguousarray(rows[:, k + 1:k + 4]), np.ascontiguousarray(rows[:, k]),
                  np.ascontiguousarray(sh.reshape(count, 48)), np.zeros(3, np.float32))
    return scene, warnings


def _camera_from_json(j: dict, index: int, warnings: list) -> Camera:
    names = {v: k for k, v in MODEL_NAMES.items()}
    try:
        model = names[j["model"]]
    except KeyError:
        raise RuntimeError(f"load_cameras: unknown camera model '{j.get('model')}'")
    w, h = int(j["width"]), int(j["height"])
    if w < 16 or h < 16:
        raise RuntimeError(f"load_cameras: camera {index}: width and height must be >= 16")
    fx = fy = cx = cy = 0.0
    if model != CAMERA_PANORAMA:
        fx, fy, cx, cy = (float(j[k]) for k in ("fx", "fy", "cx", "cy"))
        if not (fx > 0) or not (fy > 0):
            raise RuntimeError(f"load_cameras: camera {index}: focal lengths must be positive")
    fov = math.radians(float(j.get("fov_max_deg", 90.0)))
    rot, tr = list(j["rotation"]), list(j["translation"])
    if len(rot) != 9 or len(tr) != 3:
        raise RuntimeError(f"load_cameras: camera {index}: rotation needs 9 numbers (row-major) and translation 3")
    r = np.asarray(rot, np.float64).reshape(3, 3)
    dev = float(np.abs(r.T @ r - np.eye(3)).max())
    if dev > 1e-2:
        raise RuntimeError(f"load_cameras: camera {index}: rotation is not orthonormal (deviation {dev:.6f})")
    if dev > 1e-6 or np.linalg.det(r) < 0:
        u, _, vt = np.linalg.svd(r)
        fixed = u @ vt
        if np.linalg.det(fixed) < 0:
            raise RuntimeError(f"load_cameras: camera {index}: rotation has negative determinant")
        r = fixed
        warnings.append(f"load_cameras: camera {index}: rotation re-orthonormalized (deviation {dev:.6f})")
    cam = Camera(w, h, fx, fy, cx, cy, r, np.asarray(tr, np.float64), fov, model)
    return cam


def load_cameras(path: str):
    """Returns (list of Camera (float64 fields, as the reference's Camera<double>), warnings)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"load_cameras: cannot open {path}")
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise RuntimeError(f"load_cameras: {path}: {e}")
    cams = doc if isinstance(doc, list) else (doc["cameras"] if isinstance(doc, dict) and "cameras" in doc else [doc])
    warnings, out = [], []
    try:
        for i, c in enumerate(cams):
            out.append(_camera_from_json(c, i, warnings))
    except KeyError as e:
        raise RuntimeError(f"load_cameras: {path}: key {e} not found")
    if not out:
        raise RuntimeError(f"load_cameras: {path} contains no cameras")
    return out, warnings


def save_cameras(cameras, path: str) -> None:
    doc = []
    for c in cameras:
        j = {"model": MODEL_NAMES[c.model], "width": int(c.width), "height": int(c.height)}
        if c.model != CAMERA_PANORAMA:
            j.update(fx=float(c.fx), fy=float(c.fy), cx=float(c.cx), cy=float(c.cy))
        if c.model == CAMERA_FISHEYE:
            j["fov_max_deg"] = math.degrees(c.fov_max)
        j["rotation"] = [float(v) for v in np.asarray(c.rotation_wc, np.float64).reshape(9)]
        j["translation"] = [float(v) for v in np.asarray(c.translation_wc, np.float64).reshape(3)]
        doc.append(j)
    with open(path, "w") as f:
        json.dump(doc, f, indent=2)
        f.write("\n")
