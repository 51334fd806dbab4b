"""Training step on the GPU against the oracle: the L1 + D-SSIM loss and
its image gradient (inc/metrics.hpp:86-195), the Adam update (inc/optimize.hpp:100-145), their
composition in fgs_train_step, and a short optimisation that must reduce the loss.
Tolerances (fp32 device vs the fp64 reference arithmetic): loss terms rel 1e-5, image gradient
rel-L2 1e-4, Adam parameters / moments 1e-6 relative (+5e-8 absolute: fp32 parameter storage)."""
import numpy as np
import pytest

import oracle
from paper_2409_04751_b200 import Camera, RenderOptions, synthetic
from tests._helpers import rel_l2, small_fisheye, to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rast():
    from paper_2409_04751_b200 import Rasterizer

    return Rasterizer(0)


def smooth_pair(h, w, seed):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w]
    base = 0.5 + 0.4 * np.sin(xx[..., None] * np.array([0.05, 0.07, 0.03]) + yy[..., None] * np.array([0.04, 0.02, 0.06]))
    x = np.clip(base + rng.normal(0, 0.05, (h, w, 3)), 0, 1).astype(np.float32)
    y = np.clip(base + rng.normal(0, 0.05, (h, w, 3)), 0, 1).astype(np.float32)
    return x, y


@pytest.mark.parametrize("hw", [(16, 16), (37, 53), (1168, 1752)])
def test_loss_and_gradient_match_oracle(rast, hw):
    import torch
    from paper_2409_04751_b200.train import l1_dssim_loss

    x, y = smooth_pair(*hw, seed=hw[0])
    tot, l1, dssim, d = l1_dssim_loss(rast, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), 0.2)
    rt, rl1, rd, rg = oracle.l1_dssim_loss(x, y, 0.2)
    assert abs(l1 - rl1) <= 1e-5 * rl1
    assert abs(dssim - rd) <= 1e-5 * rd + 1e-7
    assert abs(tot - rt) <= 1e-5 * rt
    assert rel_l2(d.cpu().numpy(), rg) <= 1e-4


def test_loss_rejects_shape_mismatch(rast):
    import torch
    from paper_2409_04751_b200 import InvalidArgument
    from paper_2409_04751_b200.train import l1_dssim_loss

    with pytest.raises(InvalidArgument, match="dimensions differ"):
        l1_dssim_loss(rast, torch.zeros((4, 5, 3), device="cuda"), torch.zeros((5, 4, 3), device="cuda"))


def rows_from_blocks(flat, n):
    """59*N field blocks (means, rotations, log_scales, opacities, sh) -> (N, 59) rows."""
    out, off = [], 0
    for w in (3, 4, 3, 1, 48):
        out.append(flat[off:off + w * n].reshape(n, w))
        off += w * n
    return np.concatenate(out, axis=1)


@pytest.mark.parametrize("sh_rest", [0.0, 1e-4])
def test_adam_matches_oracle(rast, sh_rest):
    import torch
    from paper_2409_04751_b200.train import TrainConfig, Trainer

    sc, _, _, _ = synthetic.config(1, n=1000)
    cfg = TrainConfig(lr_sh_rest=sh_rest)
    tr = Trainer(sc, cfg, extent=2.5, rasterizer=rast)
    n = sc.n
    p_rows = rows_from_blocks(tr.params.cpu().numpy().astype(np.float64), n)
    m = np.zeros_like(p_rows)
    v = np.zeros_like(p_rows)
    lr = dict(mean=cfg.lr_mean * 2.5, rotation=cfg.lr_rotation, log_scale=cfg.lr_log_scale, opacity=cfg.lr_opacity,
              sh_dc=cfg.lr_sh_dc, sh_rest=sh_rest)
    rng = np.random.default_rng(0)
    step = 0
    for it in range(3):
        g = rng.normal(0, 1e-3, 59 * n).astype(np.float32)
        tr.adam_step(torch.from_numpy(g).cuda())
        step = oracle.adam_step(p_rows, rows_from_blocks(g.astype(np.float64), n), m, v, step, lr)
    got = rows_from_blocks(tr.params.cpu().numpy().astype(np.float64), n)
    # parameters are stored in fp32: each of the 3 updates rounds once (|step| <= lr)
    np.testing.assert_allclose(got, p_rows, rtol=1e-6, atol=5e-8)
    np.testing.assert_allclose(rows_from_blocks(tr.m.cpu().numpy().astype(np.float64), n), m, rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(rows_from_blocks(tr.v.cpu().numpy().astype(np.float64), n), v, rtol=1e-5, atol=1e-13)
    assert tr.step_count == 3


def test_adam_nonfinite_raises_without_update(rast):
    import torch
    from paper_2409_04751_b200.train import NonFinite, Trainer

    sc, _, _, _ = synthetic.config(1, n=100)
    tr = Trainer(sc, rasterizer=rast)
    before = tr.params.clone()
    g = torch.zeros(59 * 100, device="cuda")
    g[3 * 100 + 4 * 7 + 2] = float("nan")  # rotation of Gaussian 7
    with pytest.raises(NonFinite, match="non-finite gradient for Gaussian 7"):
        tr.adam_step(g)
    assert torch.equal(before, tr.params) and tr.step_count == 0


def test_train_step_is_forward_loss_backward_adam(rast):
    """fgs_train_step == Rasterizer.forward + l1_dssim_loss + backward (+ Adam), and the loss
    equals the oracle chain's (parity render + reference loss)."""
    import torch
    from paper_2409_04751_b200 import BackwardOptions
    from paper_2409_04751_b200.train import TrainConfig, Trainer, l1_dssim_loss

    sc, deg, cams, _ = synthetic.config(1, n=20000)
    cam = small_fisheye(320, 240)
    target_np = np.clip(np.random.default_rng(4).uniform(0, 0.3, (240, 320, 3)), 0, 1).astype(np.float32)
    target = torch.from_numpy(target_np).cuda()
    cfg = TrainConfig(sh_degree=3)
    tr = Trainer(sc, cfg, extent=1.0, rasterizer=rast)
    ds = to_device(sc)
    img, _ = rast.forward(ds, cam, RenderOptions(sh_degree=3))
    tot_ref, _, _, d = l1_dssim_loss(rast, img, target, cfg.loss_lambda)
    g = rast.backward(ds, cam, d, BackwardOptions(full_sh=False))
    torch.cuda.synchronize()
    res = oracle.render(sc, cam, sh_degree=3)
    ot, ol1, od, _ = oracle.l1_dssim_loss(res.image, target_np, cfg.loss_lambda)
    p0 = rows_from_blocks(tr.params.cpu().numpy().astype(np.float64), sc.n)
    total, l1, dssim = tr.step(cam, target)
    assert abs(total - tot_ref) <= 1e-7 * abs(tot_ref)  # same device path, same numbers
    assert abs(total - ot) <= 1e-5 * ot and abs(l1 - ol1) <= 1e-5 * ol1
    m = np.zeros_like(p0)
    v = np.zeros_like(p0)
    lr = dict(mean=cfg.lr_mean, rotation=cfg.lr_rotation, log_scale=cfg.lr_log_scale, opacity=cfg.lr_opacity,
              sh_dc=cfg.lr_sh_dc)
    oracle.adam_step(p0, rows_from_blocks(g.cpu().numpy().astype(np.float64), sc.n), m, v, 0, lr)
    np.testing.assert_allclose(rows_from_blocks(tr.params.cpu().numpy().astype(np.float64), sc.n), p0,
                               rtol=1e-6, atol=5e-8)


def test_short_training_reduces_loss():
    """A perturbed copy of a ground-truth scene is fitted to 8 fisheye views of it."""
    import torch
    from paper_2409_04751_b200 import Rasterizer
    from paper_2409_04751_b200.train import Dataset, TrainConfig, View, train

    gt, _, _, _ = synthetic.config(0, n=3000)
    r = Rasterizer(0)
    views = []
    for k in range(8):
        a = 2 * np.pi * k / 8
        rot = np.array([[np.cos(a), 0, -np.sin(a)], [0, 1, 0], [np.sin(a), 0, np.cos(a)]])
        cam = Camera.fisheye(128, 128, 128 / np.pi, 128 / np.pi, 64, 64)
        cam.rotation_wc = rot
        cam.translation_wc = np.zeros(3)
        cam = cam.as_float32()
        img, _ = r.forward(to_device(gt), cam, RenderOptions(sh_degree=0))
        views.append(View(cam, img.cpu().numpy()))
    init = gt.astype(np.float32)
    rng = np.random.default_rng(9)
    init.means = (init.means + rng.normal(0, 0.05, init.means.shape)).astype(np.float32)
    init.opacity_logits = (init.opacity_logits - 0.5).astype(np.float32)
    cfg = TrainConfig(iterations=120, eval_every=60, lr_mean=1e-2)
    res = train(init, Dataset(views), cfg)
    first = np.mean([row["loss"] for row in res.trace[:7]])
    last = np.mean([row["loss"] for row in res.trace[-7:]])
    assert last < 0.8 * first, (first, last)
    assert res.trace[-1]["test_psnr"] > res.trace[59]["test_psnr"] - 0.5
