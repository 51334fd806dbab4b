"""Host I/O: the reference's scene PLY / camera JSON / image formats, in
the C++ header (include/fgs_io.hpp, exercised through tools/fgs_cli) and the Python mirror
(paper_2409_04751_b200/io.py). Cases follow the reference's tests/test_io.cpp behaviour:
round trips, the DC-only layout warning, format errors, camera validation and rotation
re-orthonormalisation."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2409_04751_b200 import Camera, io, synthetic
from paper_2409_04751_b200.types import CAMERA_FISHEYE, CAMERA_PANORAMA, CAMERA_PINHOLE

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "fgs_cli")


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        from paper_2409_04751_b200.build import build_example

        build_example()
    return CLI


def run_cli(cli, *args):
    return subprocess.run([cli, *args], capture_output=True, text=True, timeout=120)


def inspect(cli, *args):
    out = run_cli(cli, "inspect", *args)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    parse = lambda ln: ({"warning": ln[len("warning="):]} if ln.startswith("warning=") else
                        dict(t.split("=", 1) for t in ln.split() if "=" in t))
    return [parse(ln) for ln in lines]


def small_scene(n=257, seed=3):
    scene, _, _, _ = synthetic.config(1, n=n)
    return scene


def test_ply_round_trip_python_and_cpp(tmp_path, cli):
    sc = small_scene()
    p = str(tmp_path / "s.ply")
    io.save_ply(sc, p)
    back, warn = io.load_ply(p)
    assert warn == []
    for f in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
        np.testing.assert_array_equal(getattr(back, f), getattr(sc, f))
    (info,) = inspect(cli, "--scene", p)
    assert int(info["gaussians"]) == sc.n
    for key, arr in (("means", sc.means), ("rotations", sc.rotations), ("log_scales", sc.log_scales),
                     ("opacity", sc.opacity_logits), ("sh", sc.sh)):
        a64 = np.asarray(arr, np.float64)
        assert abs(float(info[key]) - float(np.sum(a64))) <= 1e-12 * float(np.sum(np.abs(a64))) + 1e-30, key


def write_header(path, props, count, fmt="binary_little_endian", ptype="float"):
    with open(path, "wb") as f:
        f.write(f"ply\nformat {fmt} 1.0\nelement vertex {count}\n".encode())
        for p in props:
            f.write(f"property {ptype} {p}\n".encode())
        f.write(b"end_header\n")


def test_ply_dc_only_layout_warns_and_zeroes_rest(tmp_path, cli):
    p = str(tmp_path / "dc.ply")
    write_header(p, io.DC_PROPS, 2)
    rows = np.arange(2 * 17, dtype="<f4").reshape(2, 17)
    with open(p, "ab") as f:
        f.write(rows.tobytes())
    sc, warn = io.load_ply(p)
    assert warn == ["load_ply: f_rest_* properties missing; higher-order SH set to zero"]
    assert (sc.sh.reshape(2, 3, 16)[:, :, 1:] == 0).all()
    np.testing.assert_array_equal(sc.sh.reshape(2, 3, 16)[:, :, 0], rows[:, 6:9])
    np.testing.assert_array_equal(sc.opacity_logits, rows[:, 9])
    np.testing.assert_array_equal(sc.log_scales, rows[:, 10:13])
    np.testing.assert_array_equal(sc.rotations, rows[:, 13:17])
    infos = inspect(cli, "--scene", p)
    assert infos[0]["warning"].startswith("load_ply: f_rest_*")


@pytest.mark.parametrize("case,msg", [
    ("ascii", "binary_little_endian required, got format 'ascii'"),
    ("double", "has type 'double', expected float"),
    ("layout", "unknown property layout"),
    ("truncated", "truncated payload"),
    ("notply", "is not a PLY file"),
])
def test_ply_errors(tmp_path, cli, case, msg):
    p = str(tmp_path / f"{case}.ply")
    if case == "ascii":
        write_header(p, io.FULL_PROPS, 1, fmt="ascii")
    elif case == "double":
        write_header(p, io.FULL_PROPS, 1, ptype="double")
    elif case == "layout":
        write_header(p, io.FULL_PROPS[:-1], 1)
    elif case == "truncated":
        write_header(p, io.FULL_PROPS, 3)
        with open(p, "ab") as f:
            f.write(np.zeros(62 * 2 + 5, "<f4").tobytes())
    else:
        open(p, "w").write("not a ply\n")
    with pytest.raises(RuntimeError, match=msg):
        io.load_ply(p)
    out = run_cli(cli, "inspect", "--scene", p)
    assert out.returncode == 1 and msg in out.stderr, out.stderr


def rot(axis, ang):
    a = np.asarray(axis, np.float64) / np.linalg.norm(axis)
    k = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(ang) * k + (1 - math.cos(ang)) * k @ k


def test_camera_json_round_trip_and_models(tmp_path, cli):
    cams = [Camera(640, 480, 500.0, 501.0, 320.5, 240.25, rot([1, 2, 3], 0.7), np.array([0.1, -2, 3]),
                   math.radians(100.0), CAMERA_FISHEYE),
            Camera.pinhole(320, 240, 300.0, 300.0, 160.0, 120.0),
            Camera.panorama(1024, 512)]
    p = str(tmp_path / "c.json")
    io.save_cameras(cams, p)
    back, warn = io.load_cameras(p)
    assert warn == []
    for a, b in zip(cams, back):
        assert a.model == b.model and (a.width, a.height) == (b.width, b.height)
        np.testing.assert_allclose(b.rotation_wc, a.rotation_wc, atol=1e-15)
        np.testing.assert_allclose(b.translation_wc, a.translation_wc, atol=1e-15)
    assert math.isclose(back[0].fov_max, math.radians(100.0), rel_tol=1e-14)
    assert back[1].fov_max == math.pi / 2  # default 90 deg
    infos = inspect(cli, "--scene", _tiny_ply(tmp_path), "--cameras", p)[1:]
    assert [i["model"] for i in infos] == ["fisheye_equidistant", "pinhole", "panorama"]
    r = np.array([float(v) for v in infos[0]["rot"].split(",")]).reshape(3, 3)
    np.testing.assert_allclose(r, cams[0].rotation_wc, atol=1e-15)
    assert float(infos[0]["fx"]) == 500.0 and float(infos[0]["cy"]) == 240.25


def _tiny_ply(tmp_path):
    p = str(tmp_path / "tiny.ply")
    if not os.path.exists(p):
        io.save_ply(small_scene(4), p)
    return p


def test_camera_rotation_reorthonormalised_like_svd(tmp_path, cli):
    r = rot([0.3, -1, 0.5], 1.1) + 1e-4 * np.array([[1, 2, 0], [0, -1, 3], [2, 0, 1]])
    doc = {"cameras": [{"model": "fisheye_equidistant", "width": 64, "height": 48, "fx": 20, "fy": 20, "cx": 32,
                        "cy": 24, "rotation": list(r.reshape(9)), "translation": [0, 0, 0]}]}
    p = str(tmp_path / "r.json")
    json.dump(doc, open(p, "w"))
    cams, warn = io.load_cameras(p)
    assert len(warn) == 1 and "re-orthonormalized" in warn[0]
    u, _, vt = np.linalg.svd(r)
    np.testing.assert_allclose(cams[0].rotation_wc, u @ vt, atol=1e-12)
    infos = inspect(cli, "--scene", _tiny_ply(tmp_path), "--cameras", p)
    assert "re-orthonormalized" in infos[1]["warning"]
    w2 = infos[2]
    rc = np.array([float(v) for v in w2["rot"].split(",")]).reshape(3, 3)
    np.testing.assert_allclose(rc, u @ vt, atol=1e-12)


@pytest.mark.parametrize("cam,msg", [
    ({"model": "fisheye_equidistant", "width": 8, "height": 48, "fx": 1, "fy": 1, "cx": 0, "cy": 0,
      "rotation": [1, 0, 0, 0, 1, 0, 0, 0, 1], "translation": [0, 0, 0]}, "width and height must be >= 16"),
    ({"model": "pinhole", "width": 64, "height": 48, "fx": 0, "fy": 1, "cx": 0, "cy": 0,
      "rotation": [1, 0, 0, 0, 1, 0, 0, 0, 1], "translation": [0, 0, 0]}, "focal lengths must be positive"),
    ({"model": "orthographic", "width": 64, "height": 48}, "unknown camera model 'orthographic'"),
    ({"model": "panorama", "width": 64, "height": 48, "rotation": [1, 0, 0, 0, 1, 0, 0, 0, 1.2],
      "translation": [0, 0, 0]}, "rotation is not orthonormal"),
    ({"model": "panorama", "width": 64, "height": 48, "rotation": [1, 0, 0, 0, 1, 0], "translation": [0, 0, 0]},
     "rotation needs 9 numbers"),
])
def test_camera_errors(tmp_path, cli, cam, msg):
    p = str(tmp_path / "bad.json")
    json.dump([cam], open(p, "w"))
    with pytest.raises(RuntimeError, match=msg):
        io.load_cameras(p)
    out = run_cli(cli, "inspect", "--scene", _tiny_ply(tmp_path), "--cameras", p)
    assert out.returncode == 1 and msg in out.stderr, out.stderr
