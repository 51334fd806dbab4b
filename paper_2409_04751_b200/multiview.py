"""Multi-view batches across GPUs.

The reference renders one scene x one camera per call (inc/splatting.hpp:330-332); multi-view
work is a loop over views. Across GPUs the views are partitioned by camera with the Gaussians
replicated on every rank:
  * batched forward (config 3): view v -> rank v mod G, no collective (images stay local);
  * multi-view fwd+bwd (config 4): each rank accumulates the per-Gaussian gradients of its views
    in one 59*N buffer (fgs_backward with accumulate=1, no atomics), then ONE all-reduce(sum) of
    that buffer over NCCL (NVLink/NVSwitch). That is the only collective on the path.
"""
from __future__ import annotations

from typing import Callable, Sequence


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
