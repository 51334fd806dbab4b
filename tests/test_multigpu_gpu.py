"""The multi-GPU layer on the B200, with the CUDA kernels.

This pool gives one GPU per run, so:
* fgs_fwd_bwd_views (the native rank step) equals the sequential per-view forward / accumulating
  backward bit for bit;
* with the library's NCCL communicator at world size 1 (csrc/comm.cu: the last view's gradients
  in 4 Gaussian-id ranges, each all-reduced on a communication stream while the next range is
  computed) the result is again identical -- the chunked launch and the NCCL plumbing run for real;
* two processes on the one GPU, each rendering its half of config 4's views with the CUDA kernels,
  sum their gradients with a gloo all-reduce of the CUDA tensors: the result equals the 8-view sum
  of one process to fp32 summation order (rel-L2 <= 1e-6). (Two NCCL ranks cannot share one GPU.)
"""
import os
import socket

import numpy as np
import pytest
import torch

from tests._helpers import to_device

pytestmark = pytest.mark.gpu

N_SCENE = 400_000  # config 4's distributions at a size that keeps the 2-process test quick


def _setup(views=4, rank=0):
    from paper_2409_04751_b200 import synthetic

    scene, deg, cams, dls = synthetic.config(4, n=N_SCENE, views=views, rank=rank)
    return scene, deg, cams, dls


@pytest.fixture(scope="module")
def rast():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2409_04751_b200 import Rasterizer

    return Rasterizer(0)


def _sequential(rast, ds, deg, cams, dls_dev):
    from paper_2409_04751_b200 import BackwardOptions, RenderOptions

    g = torch.zeros(59 * ds.n, dtype=torch.float32, device="cuda")
    for v, cam in enumerate(cams):
        rast.forward(ds, cam, RenderOptions(sh_degree=deg))
        rast.backward(ds, cam, dls_dev[v], BackwardOptions(), grads=g, accumulate=v > 0)
    torch.cuda.synchronize()
    return g


def test_native_views_step_matches_sequential(rast):
    from paper_2409_04751_b200 import RenderOptions

    scene, deg, cams, dls = _setup()
    ds = to_device(scene)
    dls_dev = [torch.from_numpy(d).cuda() for d in dls]
    ref = _sequential(rast, ds, deg, cams, dls_dev)
    imgs = [torch.empty((c.height, c.width, 3), device="cuda") for c in cams]
    got = rast.fwd_bwd_views(ds, cams, dls_dev, RenderOptions(sh_degree=deg), images=imgs)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    # the images are the per-view forwards
    one = rast.forward(ds, cams[2], RenderOptions(sh_degree=deg))[0]
    assert torch.equal(one, imgs[2])


def test_nccl_one_rank_chunked_allreduce(rast):
    from paper_2409_04751_b200 import RenderOptions
    from paper_2409_04751_b200.multiview import Communicator

    scene, deg, cams, dls = _setup()
    ds = to_device(scene)
    dls_dev = [torch.from_numpy(d).cuda() for d in dls]
    ref = rast.fwd_bwd_views(ds, cams, dls_dev, RenderOptions(sh_degree=deg)).clone()
    comm = Communicator(rast, Communicator.unique_id(), 1, 0)
    try:
        got = rast.fwd_bwd_views(ds, cams, dls_dev, RenderOptions(sh_degree=deg), comm=comm)
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
        again = comm.allreduce(got.clone(), scene.n)
        torch.cuda.synchronize()
        assert torch.equal(again, ref)
        # no views on this rank: it contributes zeros
        z = rast.fwd_bwd_views(ds, [], [], RenderOptions(sh_degree=deg), grads=torch.ones_like(ref), comm=comm)
        torch.cuda.synchronize()
        assert not z.any()
    finally:
        comm.close()


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_2409_04751_b200 import Rasterizer, RenderOptions, multiview

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, deg, cams, dls = _setup(views=8)
    mine = multiview.partition_views(len(cams), world, rank)
    r = Rasterizer(0)
    ds = to_device(scene)
    g = r.fwd_bwd_views(ds, [cams[v] for v in mine], [torch.from_numpy(dls[v]).cuda() for v in mine],
                        RenderOptions(sh_degree=deg))
    torch.cuda.synchronize()
    dist.all_reduce(g, op=dist.ReduceOp.SUM)  # gloo over the CUDA tensor
    if rank == 0:
        np.save(out_path, g.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_process_cuda_gradient_sum(rast, tmp_path):
    import torch.multiprocessing as mp

    from paper_2409_04751_b200 import RenderOptions

    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out).astype(np.float64)
    scene, deg, cams, dls = _setup(views=8)
    ds = to_device(scene)
    single = rast.fwd_bwd_views(ds, cams, [torch.from_numpy(d).cuda() for d in dls], RenderOptions(sh_degree=deg))
    ref = single.double().cpu().numpy()
    assert np.abs(ref).sum() > 0
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 1e-6, rel
