"""The training-step oracle pinned to the reference's own code: the numpy
restatements of l1_dssim_loss (inc/metrics.hpp:86-195) and adam_step (inc/optimize.hpp:100-145)
against the reference headers compiled in oracle/_ref."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="reference build (oracle/_ref) absent")


@pytest.mark.parametrize("shape", [(16, 16), (37, 53), (64, 48)])
def test_l1_dssim_loss_matches_reference(shape):
    rng = np.random.default_rng(sum(shape))
    x = rng.uniform(0, 1, shape + (3,))
    y = np.clip(x + rng.normal(0, 0.1, x.shape), 0, 1)
    for lam in (0.2, 0.0, 1.0):
        a = oracle.l1_dssim_loss(x, y, lam)
        b = oracle.ref_l1_dssim_loss(x, y, lam)
        np.testing.assert_allclose(a[:3], b[:3], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(a[3], b[3], rtol=1e-10, atol=1e-16)


def test_ssim_of_identical_images_is_one_with_zero_gradient():  # metrics.hpp:121-124
    x = np.random.default_rng(1).uniform(0, 1, (20, 30, 3))
    total, l1, dssim, d = oracle.ref_l1_dssim_loss(x, x, 0.2)
    assert l1 == 0 and abs(dssim) < 1e-12 and np.abs(d).max() == 0
    s, g = oracle.ssim(x, x, want_grad=True)
    assert abs(s - 1) < 1e-12 and np.abs(g).max() == 0


def test_adam_step_matches_reference():
    rng = np.random.default_rng(2)
    n = 17
    p = rng.normal(size=(n, 59))
    m = np.zeros((n, 59))
    v = np.zeros((n, 59))
    lr = dict(mean=1.6e-4 * 3.0, rotation=1e-3, log_scale=5e-3, opacity=5e-2, sh_dc=2.5e-3)
    p1, m1, v1 = p.copy(), m.copy(), v.copy()
    p2, m2, v2 = p.copy(), m.copy(), v.copy()
    s1 = s2 = 0
    for it in range(4):
        g = rng.normal(size=(n, 59))
        s1 = oracle.adam_step(p1, g, m1, v1, s1, lr)
        s2 = oracle.ref_adam_step(p2, g, m2, v2, s2, lr)
        np.testing.assert_allclose(p1, p2, rtol=0, atol=1e-15)
        np.testing.assert_allclose(m1, m2, rtol=0, atol=1e-15)
        np.testing.assert_allclose(v1, v2, rtol=0, atol=1e-15)
    assert s1 == s2 == 4
    rest = oracle.PARAM_GROUPS["sh_rest"]
    np.testing.assert_array_equal(p1[:, rest], p[:, rest])  # the reference leaves bands 1..3 alone
