"""The restatement (libm mode) against the reference build (oracle/_ref) on fresh seeded
scenes: every forward field and the DC-only gradients must be bit-identical; all three camera
models, SH degrees 0-3, rotated poses. Skipped when oracle/_ref is absent."""
import math

import numpy as np
import pytest

import oracle
from paper_2409_04751_b200 import Camera, synthetic
from tests.golden.make_golden import spherical_scene

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def cameras():
    yield Camera.fisheye(128, 96, 30.0, 30.0, 64.0, 48.0)
    yield Camera.pinhole(128, 96, 80.0, 80.0, 64.0, 48.0)
    yield Camera.panorama(128, 64)
    c = Camera.fisheye(160, 120, 35.0, 33.0, 81.0, 59.0, math.radians(95))
    c.rotation_wc, c.translation_wc = synthetic.random_pose(np.random.default_rng(9), box=0.5)
    yield c


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_bit_exact_vs_reference(deg, dtype):
    scene = spherical_scene(600, 40 + deg)
    for cam in cameras():
        cam = cam.as_float32()
        a = oracle.render(scene, cam, sh_degree=deg, dtype=dtype, mode=oracle.MODE_LIBM)
        b = oracle.render(scene, cam, sh_degree=deg, dtype=dtype, impl="ref")
        for f in ("mean_px", "conic", "depth", "radius", "color", "alpha", "source", "refs", "offsets", "image",
                  "cam_points"):
            assert a.get(f).tobytes() == b.get(f).tobytes(), (f, cam.model)
        dl = np.random.default_rng(deg).standard_normal((cam.height, cam.width, 3))
        ga, sa = oracle.backward(a, scene.n, dl, full_sh=False, mode=oracle.MODE_LIBM, want_splat_grads=True)
        gb, sb = oracle.backward(b, scene.n, dl, want_splat_grads=True)
        assert ga.tobytes() == gb.tobytes() and sa.tobytes() == sb.tobytes(), cam.model


def test_bruteforce_matches_reference():
    scene = spherical_scene(150, 3)
    cam = Camera.fisheye(96, 80, 28.0, 28.0, 48.0, 40.0)
    a, _ = oracle.bruteforce_render(scene, cam, sh_degree=3)
    b, _ = oracle.bruteforce_render(scene, cam, sh_degree=3, impl="ref")
    assert np.abs(a - b).max() < 1e-12


def test_zero_quaternion_error_matches_reference():
    scene = spherical_scene(50, 1)
    scene.rotations[7] = 0
    cam = Camera.fisheye(96, 80, 28.0, 28.0, 48.0, 40.0)
    with pytest.raises(oracle.OracleError, match="degenerate rotation"):
        oracle.render(scene, cam, impl="ref")
    with pytest.raises(oracle.OracleError, match="degenerate rotation"):
        oracle.render(scene, cam)
