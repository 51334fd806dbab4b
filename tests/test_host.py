"""Host-side logic without a GPU: synthetic workloads, camera/option conversion, gradient
buffer layout, reference error behaviour on the Python side."""
import math

import numpy as np
import pytest

from paper_2409_04751_b200 import BackwardOptions, Camera, RenderOptions, split_grads, synthetic
from paper_2409_04751_b200.api import GRAD_FIELDS, InvalidArgument, _backward_options, _camera_struct, grads_as_rows


def test_synthetic_configs_are_seeded_and_shaped():
    a, deg, cams, dls = synthetic.config(0)
    b, _, _, _ = synthetic.config(0)
    assert deg == 0 and a.n == 10_000 and a.sh.shape == (10_000, 48)
    assert np.array_equal(a.means, b.means) and a.means.dtype == np.float32
    r = np.linalg.norm(a.means, axis=1)
    assert r.min() >= 1.0 - 1e-5 and r.max() <= 10.0 + 1e-5
    assert not a.sh[:, [k for k in range(48) if k % 16]].any()  # SH degree 0: bands 1-3 zero
    cam = cams[0]
    assert (cam.width, cam.height) == (256, 256) and cam.fx == pytest.approx(256 / math.pi, rel=1e-6)
    s1, deg1, cams1, dls1 = synthetic.config(1, n=1000)
    assert deg1 == 3 and dls1[0].shape == (1168, 1752, 3)
    assert cams1[0].fx == pytest.approx(670.247, rel=1e-5)
    s3, _, cams3, _ = synthetic.config(3, n=1000)
    assert len(cams3) == 64 and cams3[0].fov_max == pytest.approx(math.radians(95), rel=1e-6)
    R = cams3[5].rotation_wc
    np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-6)


def test_camera_struct_roundtrip_and_equality():
    cam = synthetic.fisheye_full()
    c = _camera_struct(cam)
    assert (c.width, c.height, c.model) == (1752, 1168, 1)
    assert c.fx == np.float32(cam.fx)
    other = Camera(**{**cam.__dict__})
    assert cam.same_as(other)
    other.fx += 1.0
    assert not cam.same_as(other)


def test_gradient_buffer_layout():
    n = 5
    buf = np.arange(59 * n, dtype=np.float32)
    s = split_grads(buf, n)
    assert s["mean"].shape == (n, 3) and s["sh"].shape == (n, 48) and s["opacity"].shape == (n,)
    assert s["rotation"][0, 0] == 3 * n and s["sh"][0, 0] == 11 * n
    rows = grads_as_rows(buf, n)
    assert rows.shape == (n, 59) and rows[1, 0] == 3 and rows[0, 10] == 10 * n
    assert sum(k for _, k in GRAD_FIELDS) == 59


def test_backward_options_defaults_match_reference():
    o = _backward_options(BackwardOptions(), accumulate=False)
    assert list(o.jacobian_grad_scale) == [1.0, 1.0, 1.0]
    assert o.full_sh == 1 and o.accumulate == 0 and o.sh_view_dir_grad == 0
