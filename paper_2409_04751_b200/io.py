"""Python mirror of the host I/O in include/fgs_io.hpp: the reference's scene PLY and camera
JSON formats.

  load_ply / save_ply          the format of src/ply_io.cpp:40-145 (3DGS binary_little_endian layout)
  load_cameras / save_cameras  the format of src/camera_io.cpp:25-127

Only the formats and the error messages follow the reference; the readers are schema-driven
(one (name, field, component) column per PLY property), as in include/fgs_io.hpp.

Errors are RuntimeError with the reference's messages; warnings are returned, as the
reference's PlyReadResult / CameraReadResult do.
"""
from __future__ import annotations

import json
import math

import numpy as np

from .types import CAMERA_FISHEYE, CAMERA_PANORAMA, CAMERA_PINHOLE, Camera, Scene

def _ply_schema(with_rest: bool):
    """Vertex properties of the 3DGS PLY layout as (name, field, component) columns -- the
    schema of include/fgs_io.hpp's reader. SH components index the scene's [channel*16 + basis]
    row; the file keeps f_rest_{c*15 + j - 1} for basis j >= 1 of channel c."""
    cols = [(a, "mean", k) for k, a in enumerate("xyz")] + [("n" + a, None, k) for k, a in enumerate("xyz")]
    cols += [(f"f_dc_{c}", "sh", 16 * c) for c in range(3)]
    if with_rest:
        cols += [(f"f_rest_{r}", "sh", 16 * (r // 15) + r % 15 + 1) for r in range(45)]
    cols += [("opacity", "opacity", 0)] + [(f"scale_{k}", "log_scale", k) for k in range(3)]
    cols += [(f"rot_{k}", "rotation", k) for k in range(4)]
    return cols


FULL_PROPS = [c[0] for c in _ply_schema(True)]
DC_PROPS = [c[0] for c in _ply_schema(False)]
MODEL_NAMES = {CAMERA_PINHOLE: "pinhole", CAMERA_FISHEYE: "fisheye_equidistant", CAMERA_PANORAMA: "panorama"}
_WIDTH = {"mean": 3, "sh": 48, "opacity": 1, "log_scale": 3, "rotation": 4}


def _scene_fields(scene: Scene) -> dict:
    return {"mean": np.asarray(scene.means, np.float32).reshape(-1, 3),
            "sh": np.asarray(scene.sh, np.float32).reshape(-1, 48),
            "opacity": np.asarray(scene.opacity_logits, np.float32).reshape(-1, 1),
            "log_scale": np.asarray(scene.log_scales, np.float32).reshape(-1, 3),
            "rotation": np.asarray(scene.rotations, np.float32).reshape(-1, 4)}


def save_ply(scene: Scene, path: str) -> None:
    schema = _ply_schema(True)
    fields = _scene_fields(scene)
    block = np.zeros((scene.n, len(schema)), "<f4")
    for col, (_, field, comp) in enumerate(schema):
        if field is not None:
            block[:, col] = fields[field][:, comp]
    head = f"ply\nformat binary_little_endian 1.0\nelement vertex {scene.n}\n"
    head += "".join(f"property float {name}\n" for name, _, _ in schema) + "end_header\n"
    with open(path, "wb") as f:
        f.write(head.encode())
        f.write(block.tobytes())


def _read_ply_header(f, path):
    """(vertex count, property names, payload offset); raises with the reference's messages."""
    def line():
        raw = f.readline()
        return None if not raw else raw.decode("latin1").rstrip("\n").rstrip("\r")

    if line() != "ply":
        raise RuntimeError(f"load_ply: {path} is not a PLY file")
    count, fmt_seen, props = 0, False, []
    while True:
        ln = line()
        if ln is None or ln == "end_header":
            break
        w = ln.split() + ["", "", ""]
        key, a1, a2 = w[0], w[1], w[2]
        if key in ("", "comment", "obj_info"):
            continue
        if key == "format":
            if a1 != "binary_little_endian":
                raise RuntimeError(f"load_ply: binary_little_endian required, got format '{a1}'")
            fmt_seen = True
        elif key == "element":
            if a1 != "vertex":
                raise RuntimeError(f"load_ply: unsupported element '{a1}'")
            count = int(a2 or 0)
        elif key == "property":
            if a1 != "float":
                raise RuntimeError(f"load_ply: property '{a2}' has type '{a1}', expected float")
            props.append(a2)
        else:
            raise RuntimeError(f"load_ply: unexpected header line '{ln}'")
    if not fmt_seen:
        raise RuntimeError("load_ply: missing format line (binary_little_endian required)")
    return count, props, f.tell()


def load_ply(path: str):
    """Returns (Scene, warnings)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"load_ply: cannot open {path}")
    with f:
        count, props, start = _read_ply_header(f, path)
        warnings, schema = [], None
        for rest in (True, False):
            if props == [c[0] for c in _ply_schema(rest)]:
                schema = _ply_schema(rest)
                if not rest:
                    warnings.append("load_ply: f_rest_* properties missing; higher-order SH set to zero")
                break
        if schema is None:
            raise RuntimeError("load_ply: unknown property layout; expected [" + ",".join(FULL_PROPS) +
                               "] (or the f_rest-free variant), found [" + ",".join(props) + "]")
        want = count * len(schema) * 4
        data = f.read(want)
    if len(data) != want:
        raise RuntimeError(f"load_ply: truncated payload at byte offset {start + len(data)}")
    block = np.frombuffer(data, "<f4").reshape(count, len(schema))
    out = {k: np.zeros((count, w), np.float32) for k, w in _WIDTH.items()}
    for col, (_, field, comp) in enumerate(schema):
        if field is not None:
            out[field][:, comp] = block[:, col]
    scene = Scene(out["mean"], out["rotation"], out["log_scale"], np.ascontiguousarray(out["opacity"][:, 0]),
                  out["sh"], np.zeros(3, np.float32))
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
