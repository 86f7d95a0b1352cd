"""Collective wrappers over torch.distributed groups (NCCL over NVLink on B200).

Every wrapper is a no-op for single-rank groups, so a layer's code path is the
same for tp=1/dp=1 and for sharded strategies.  These are the runtime's
realizations of the cost model's collective terms (costmodel.py:108-118, 199-213):
TP all-reduce / SP all-gather + reduce-scatter, ZeRO gathers and reduce-scatters,
DP all-reduce.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def all_reduce(t: torch.Tensor, g, op=dist.ReduceOp.SUM) -> torch.Tensor:
    if g is not None and g.size > 1:
        dist.all_reduce(t, op=op, group=g.group)
    return t


def all_gather(t: torch.Tensor, g, out: torch.Tensor | None = None) -> torch.Tensor:
    """Concatenate rank chunks along dim 0."""
    if g is None or g.size == 1:
        return t if out is None else out.copy_(t)
    if out is None:
        out = torch.empty((t.shape[0] * g.size,) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
    dist.all_gather_into_tensor(out, t.contiguous(), group=g.group)
    return out


def all_gather_async(t: torch.Tensor, g):
    """all_gather launched on NCCL's stream: (out, work); work.wait() orders the current
    stream after it (None work for single-rank groups)."""
    if g is None or g.size == 1:
        return t, None
    out = torch.empty((t.shape[0] * g.size,) + tuple(t.shape[1:]), dtype=t.dtype,
                      device=t.device)
    work = dist.all_gather_into_tensor(out, t.contiguous(), group=g.group, async_op=True)
    return out, work


def reduce_scatter(t: torch.Tensor, g, out: torch.Tensor | None = None) -> torch.Tensor:
    """Sum over ranks, keep this rank's dim-0 chunk."""
    if g is None or g.size == 1:
        return t if out is None else out.copy_(t)
    if out is None:
        out = torch.empty((t.shape[0] // g.size,) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
    dist.reduce_scatter_tensor(out, t.contiguous(), group=g.group)
    return out


def all_to_all(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, g) -> torch.Tensor:
    if g is None or g.size == 1:
        return out.copy_(inp)
    dist.all_to_all_single(out, inp, output_split_sizes=list(out_splits),
                           input_split_sizes=list(in_splits), group=g.group)
    return out
