"""World-size-2 CPU test (gloo) of the multi-view gradient path (config 4 logic): per-rank view
partition, per-view accumulation into one 59*N buffer, one all-reduce(sum). The per-view
render+backward is the CPU oracle here (no GPU in CI); on B200 it is fgs_backward."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_04751_b200 import multiview, synthetic
from paper_2409_04751_b200.types import Camera


def _cams_and_dls(num_views):
    rng = np.random.default_rng(11)
    cams, dls = [], []
    for _ in range(num_views):
        r_wc, t_wc = synthetic.random_pose(rng, box=2.0)
        c = Camera.fisheye(64, 48, 20.0, 20.0, 32.0, 24.0)
        c.rotation_wc, c.translation_wc = r_wc, t_wc
        cams.append(c.as_float32())
        dls.append(rng.standard_normal((48, 64, 3)).astype(np.float32))
    return cams, dls


def _scene():
    scene, _, _, _ = synthetic.config(3, n=3000)
    scene.means = (scene.means / 4.0).astype(np.float32)
    scene.log_scales = (scene.log_scales + 1.5).astype(np.float32)
    return scene


def _oracle_view_grads(scene, cam, dl):
    import oracle

    res = oracle.render(scene, cam, sh_degree=3)
    g, _ = oracle.backward(res, scene.n, dl)  # rows: (n, 59)
    from paper_2409_04751_b200.api import GRAD_FIELDS

    # to the flat field-major layout the C ABI writes
    parts, col = [], 0
    for _, k in GRAD_FIELDS:
        parts.append(g[:, col:col + k].reshape(-1))
        col += k
    return np.concatenate(parts)


def _worker(rank, world, port, num_views, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene = _scene()
    cams, dls = _cams_and_dls(num_views)
    mine = multiview.partition_views(num_views, world, rank)
    grads = torch.zeros(59 * scene.n, dtype=torch.float32)

    def render_backward(v, buf, accumulate):
        g = torch.from_numpy(_oracle_view_grads(scene, cams[v], dls[v]))
        if accumulate:
            buf += g
        else:
            buf.copy_(g)

    multiview.fwd_bwd_views(mine, render_backward, grads, process_group=dist.group.WORLD)
    if rank == 0:
        np.save(out_path, grads.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_views_covers_all():
    for views in (1, 7, 64):
        for world in (1, 2, 3, 8):
            got = sorted(v for r in range(world) for v in multiview.partition_views(views, world, r))
            assert got == list(range(views))


def test_two_rank_gradient_allreduce(tmp_path):
    import oracle

    oracle.build()
    num_views = 4
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(2, _free_port(), num_views, out), nprocs=2, join=True)
    got = np.load(out)
    scene = _scene()
    cams, dls = _cams_and_dls(num_views)
    ref = sum(_oracle_view_grads(scene, cams[v], dls[v]).astype(np.float64) for v in range(num_views))
    assert np.abs(ref).sum() > 0
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel < 1e-6, rel
