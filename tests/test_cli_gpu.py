"""The reference-compatible CLI on the GPU: `render` writes the frames
and the reference's per-frame stats line (src/cli.cpp:56-65, :125-136); `bench` prints the
reference's per-camera throughput line (src/cli.cpp:138-170). Images equal the Python API's
render of the same PLY, quantised like the reference's writer (round half to even)."""
import os
import subprocess

import numpy as np
import pytest

from paper_2409_04751_b200 import Camera, io, synthetic

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "fgs_cli")


def read_ppm(path):
    data = open(path, "rb").read()
    parts = data.split(b"\n", 3)
    assert parts[0] == b"P6"
    w, h = map(int, parts[1].split())
    return np.frombuffer(parts[3], np.uint8).reshape(h, w, 3)


def parse(line):
    return dict(t.split("=", 1) for t in line.split() if "=" in t)


@pytest.fixture(scope="module")
def dataset(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli")
    scene, deg, cams, _ = synthetic.config(1, n=20000)
    pin = Camera.pinhole(640, 480, 400.0, 400.0, 320.0, 240.0)
    io.save_ply(scene, str(d / "scene.ply"))
    io.save_cameras([cams[0], pin], str(d / "cameras.json"))
    return d, scene, [cams[0], pin]


def test_cli_render_matches_api(dataset, oracle_mod):
    import torch
    from paper_2409_04751_b200 import Rasterizer, RenderOptions
    from tests._helpers import to_device

    d, scene, cams = dataset
    out = subprocess.run([CLI, "render", "--scene", str(d / "scene.ply"), "--cameras", str(d / "cameras.json"),
                          "--out", str(d / "frames"), "--format", "ppm"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [parse(ln) for ln in out.stdout.strip().splitlines()]
    assert len(lines) == 2
    r = Rasterizer(0)
    for i, (ln, cam) in enumerate(zip(lines, cams)):
        assert ln["frame"] == str(i) and ln["model"] == ("fisheye_equidistant" if i == 0 else "pinhole")
        camf = cam.as_float32()
        img, st = r.forward(to_device(scene), camf, RenderOptions(sh_degree=3), want_stats=True)
        torch.cuda.synchronize()
        expect = np.rint(np.clip(img.cpu().numpy().astype(np.float64), 0, 1) * 255).astype(np.uint8)
        got = read_ppm(ln["file"])
        np.testing.assert_array_equal(got, expect)
        res = oracle_mod.render(scene, camf, sh_degree=3)
        assert int(ln["intersections"]) == res.num_intersections
        assert int(ln["splats"]) == res.num_splats and int(ln["culled"]) + int(ln["degenerate"]) + \
            int(ln["splats"]) == scene.n


def test_cli_bench_line(dataset):
    d, scene, cams = dataset
    out = subprocess.run([CLI, "bench", "--scene", str(d / "scene.ply"), "--cameras", str(d / "cameras.json"),
                          "--repeat", "5"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [parse(ln) for ln in out.stdout.strip().splitlines()]
    assert [ln["camera"] for ln in lines] == ["0", "1"]
    for ln in lines:
        assert ln["repeats"] == "5" and float(ln["fps"]) > 0 and int(ln["intersections"]) > 0
