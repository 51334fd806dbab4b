"""Multi-view batches across GPUs.

The reference renders one scene x one camera per call (inc/splatting.hpp:330-332); multi-view
work is a loop over views. Across GPUs the views are partitioned by camera with the Gaussians
replicated on every rank:
  * batched forward (config 3): view v -> rank v mod G, no collective (images stay local);
  * multi-view fwd+bwd (config 4): each rank accumulates the per-Gaussian gradients of its views
    in one 59*N buffer (fgs_backward with accumulate=1, no atomics), then ONE all-reduce(sum) of
    that buffer over NCCL (NVLink/NVSwitch). That is the only collective on the path.

The library does the whole rank step natively (fgs_fwd_bwd_views, csrc/comm.cu) with its own NCCL
communicator (``Communicator``), overlapping the all-reduce with the last view's preprocess
backward; ``fwd_bwd_views`` below is the same step through torch.distributed (any backend, e.g.
gloo for CPU tests).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Sequence

from . import _lib


def partition_views(num_views: int, world_size: int, rank: int) -> list:
    """View indices owned by ``rank``: v mod world_size == rank."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank / world size")
    return list(range(rank, num_views, world_size))


def forward_views(views: Sequence, render: Callable) -> list:
    """Batched forward of this rank's views; ``render(view)`` returns the image."""
    return [render(v) for v in views]


def fwd_bwd_views(views: Sequence, render_backward: Callable, grads, process_group=None, all_reduce: bool = True):
    """Forward+backward of this rank's views, summing gradients into ``grads``.

    ``render_backward(view, grads, accumulate)`` runs one view's forward and backward and writes
    (accumulate=False, first view) or adds (accumulate=True) its per-Gaussian gradients into
    ``grads``. With a process group of size > 1 the summed buffer is all-reduced once.
    """
    if len(views) == 0:
        grads.zero_() if hasattr(grads, "zero_") else grads.fill(0)
    for i, v in enumerate(views):
        render_backward(v, grads, i > 0)
    if all_reduce and process_group is not None:
        import torch.distributed as dist

        if dist.get_world_size(process_group) > 1:
            dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=process_group)
    return grads


class Communicator:
    """The library's NCCL communicator (fgs_comm) of one rank, bound to a Rasterizer's device and
    stream. ``from_process_group`` shares the NCCL id over an existing torch.distributed group."""

    def __init__(self, rasterizer, unique_id: bytes, world_size: int, rank: int):
        self._L = _lib.load()
        self._h = C.c_void_p()
        uid = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        rasterizer._check(self._L.fgs_comm_init(rasterizer._h, uid, int(world_size), int(rank), C.byref(self._h)))
        self.world_size, self.rank = world_size, rank

    @staticmethod
    def unique_id() -> bytes:
        L = _lib.load()
        buf = (C.c_uint8 * 128)()
        if L.fgs_comm_get_unique_id(buf) != _lib.FGS_OK:
            raise RuntimeError("fgs_comm_get_unique_id failed (NCCL unavailable?)")
        return bytes(buf)

    @classmethod
    def from_process_group(cls, rasterizer, group=None):
        import torch.distributed as dist

        obj = [cls.unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(rasterizer, obj[0], dist.get_world_size(group), dist.get_rank(group))

    def allreduce(self, grads, n: int):
        from .api import _grad_struct

        gs = _grad_struct(grads, n)
        rc = self._L.fgs_allreduce_gradients(self._h, C.byref(gs), int(n))
        if rc != _lib.FGS_OK:
            raise RuntimeError(f"fgs_allreduce_gradients failed with status {rc}")
        return grads

    def close(self):
        if self._h:
            self._L.fgs_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
