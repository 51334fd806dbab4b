"""Fixtures produced by the reference itself (tests/golden/make_golden.py runs the reference's
hot-path headers via oracle/_ref). The oracle restatement must reproduce them bit for bit in
libm mode; in parity mode (the GPU's transcendental definition) within tolerance; the GPU path
within the north-star tolerances."""
import glob
import os

import numpy as np
import pytest

import oracle
from paper_2409_04751_b200 import Camera, Scene
from tests._helpers import psnr, rel_l2
from tests.golden.make_golden import golden_dl

FIXTURES = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
FIELDS = ("mean_px", "conic", "depth", "radius", "color", "alpha", "source", "refs", "offsets")


def load(path):
    z = np.load(path)
    scene = Scene(z["means"], z["rotations"], z["log_scales"], z["opacity_logits"], z["sh"], z["background"])
    a = z["camera"]
    cam = Camera(int(a[1]), int(a[2]), a[3], a[4], a[5], a[6], a[7:16].reshape(3, 3), a[16:19], a[19], int(a[0]))
    return z, scene, cam, int(z["sh_degree"])


@pytest.fixture(scope="module", autouse=True)
def _build():
    oracle.build()


def test_fixtures_present():
    assert len(FIXTURES) >= 3


@pytest.mark.parametrize("path", FIXTURES, ids=lambda p: os.path.basename(p)[:-4])
def test_restatement_bit_exact_vs_reference(path):
    z, scene, cam, deg = load(path)
    res = oracle.render(scene, cam, sh_degree=deg, mode=oracle.MODE_LIBM)
    for f in FIELDS:
        got, ref = res.get(f), z[f]
        assert got.shape == ref.shape and got.tobytes() == ref.tobytes(), f
    assert res.image.tobytes() == z["image"].tobytes()
    grads, sg = oracle.backward(res, scene.n, golden_dl(cam), full_sh=False, mode=oracle.MODE_LIBM,
                                want_splat_grads=True)
    assert grads.tobytes() == z["grads"].tobytes()
    assert sg.tobytes() == z["splat_grads"].tobytes()


@pytest.mark.parametrize("path", FIXTURES, ids=lambda p: os.path.basename(p)[:-4])
def test_parity_mode_close_to_reference(path):
    z, scene, cam, deg = load(path)
    res = oracle.render(scene, cam, sh_degree=deg, mode=oracle.MODE_PARITY)
    assert np.abs(res.image.astype(np.float64) - z["image"]).max() <= 1e-3
    grads, _ = oracle.backward(res, scene.n, golden_dl(cam), full_sh=False)
    assert rel_l2(grads, z["grads"]) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=lambda p: os.path.basename(p)[:-4])
def test_gpu_vs_reference_fixture(path):
    import torch

    from paper_2409_04751_b200 import BackwardOptions, Rasterizer, RenderOptions, grads_as_rows
    from tests._helpers import to_device

    z, scene, cam, deg = load(path)
    r = Rasterizer(0)
    ds = to_device(scene)
    img, st = r.forward(ds, cam.as_float32(), RenderOptions(sh_degree=deg, background=scene.background),
                        want_stats=True)
    g = r.backward(ds, cam.as_float32(), torch.from_numpy(golden_dl(cam)).cuda(), BackwardOptions(full_sh=False))
    torch.cuda.synchronize()
    img = img.cpu().numpy()
    assert np.abs(img.astype(np.float64) - z["image"]).max() <= 1e-3
    assert psnr(img, z["image"]) >= 60.0
    assert st.num_intersections == int(z["stats"][0]) and st.num_splats == int(z["stats"][1])
    np.testing.assert_array_equal(r.debug("offsets"), z["offsets"])
    np.testing.assert_array_equal(r.debug("sorted_gauss"), z["source"][z["refs"]])
    assert rel_l2(grads_as_rows(g, scene.n), z["grads"]) <= 1e-3
