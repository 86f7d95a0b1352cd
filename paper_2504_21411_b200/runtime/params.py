"""Flat per-layer parameter / gradient / optimizer storage with ZeRO-0..3 on the dp axis.

One ``ParamStore`` per decoder layer (and one each for the embedding and the head)
holds the layer's TP-local tensors packed into one flat buffer (each entry 64-element
aligned so every GEMM operand is TMA-aligned), padded so it splits into ``dp`` equal
contiguous shards.  Memory per device follows the reference cost model exactly
(costmodel.py:157-160): params bpp*P/tp (/dp if z3), grads bpg*P/tp (/dp if z>=2),
fp32 master + Adam moments 12*P/tp (/dp if z>=1).

Communication (costmodel.py:114-118, 199-213):
  z0: grad all-reduce over dp at sync
  z1: grad reduce-scatter at sync, param all-gather after the step
  z2: grad reduce-scatter after every microbatch (shard accumulators), param AG after step
  z3: as z2, params live sharded and are all-gathered before each fwd and each bwd
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist

from .. import kernels as K
from . import comm


# bounded window of stores with reduce-scatters in flight (each holds a full-size temporary
# gradient until drained, so an unbounded window would cost one layer's grads per layer)
_INFLIGHT: "collections.deque" = None
MAX_INFLIGHT = 2


def _track(store) -> None:
    global _INFLIGHT
    import collections
    if _INFLIGHT is None:
        _INFLIGHT = collections.deque()
    _INFLIGHT.append(store)
    while len(_INFLIGHT) > MAX_INFLIGHT:
        _INFLIGHT.popleft().drain()


def _async(fn, *args, **kw):
    """Launch a torch.distributed collective asynchronously (None for single-rank groups)."""
    return fn(*args, async_op=True, **kw)

ALIGN = 64

# Timing-only switch for the profiler's dp-sync exposure measurement
# (profiler.measure_dp_overlap): when True, every dp gradient reduction and parameter
# all-gather of ZeRO-0/1/2 is skipped (each rank updates its own shard from its local
# gradients).  The numbers are wrong by construction; never set it for training.
SKIP_DP_SYNC = False


def _roundup(x: int, m: int) -> int:
    return (x + m - 1) // m * m


class ParamStore:
    def __init__(self, entries, *, dtype, grad_dtype, device, dp, zero: int,
                 small_names=(), extra_allreduce=None):
        """entries: ordered list of (name, local_shape)."""
        self.dtype, self.grad_dtype, self.device = dtype, grad_dtype, device
        # group whose members hold token-partial grads of replicated weights (Ulysses)
        self.extra = extra_allreduce
        self.dp = dp                          # GroupHandle or None
        self.ndp = dp.size if dp is not None else 1
        self.rank_dp = dp.index if dp is not None else 0
        self.zero = zero if self.ndp > 1 else 0
        self.layout = {}
        off = 0
        for name, shape in entries:
            n = math.prod(shape)
            self.layout[name] = (off, tuple(shape))
            off = _roundup(off + n, ALIGN)
        self.numel = sum(math.prod(s) for _, s in self.layout.values())
        self.total = _roundup(max(off, 1), self.ndp * ALIGN)
        self.shard = self.total // self.ndp
        self.lo = self.rank_dp * self.shard
        kw = dict(device=device)
        if self.zero == 3:
            self.p_shard = torch.zeros(self.shard, dtype=dtype, **kw)
            self.p_full = None
        else:
            self.p_full = torch.zeros(self.total, dtype=dtype, **kw)
        if self.zero >= 2:
            self.g_shard = torch.zeros(self.shard, dtype=grad_dtype, **kw)
            self.g_full = None
        else:
            self.g_full = torch.zeros(self.total, dtype=grad_dtype, **kw)
            self.g_shard = None
        # fp32 accumulators for small (1-D) entries: norms and biases
        self.small = [n for n in small_names if n in self.layout]
        self.small_layout = {}
        soff = 0
        for n in self.small:
            size = math.prod(self.layout[n][1])
            self.small_layout[n] = (soff, self.layout[n][1])
            soff += size
        self.acc32 = torch.zeros(max(soff, 1), dtype=torch.float32, **kw)
        self.master = self.m = self.v = None
        self._gathered = None
        self._gather_work = None
        self._owned_grad = None
        # overlap state: collectives in flight on NCCL streams, drained before use
        self.pending: list = []       # (work, finalize callback, keep-alive refs)
        self.last_window = False      # set by the engine for the last microbatch's backward
        self._synced = False
        self._param_ag = None
        self.ready_event = None       # optimizer update (side stream) done -> params usable
        self.nvl = None               # dp_nvlink.DpPool holding this store's flat buffers
        self._slot = None             # z2 grad-target ring slot of the current microbatch
        self._param_epoch = None      # channel-1 epoch of the peers' parameter broadcast

    def attach_nvlink(self, pool) -> None:
        """Move the full param / grad buffers into the dp group's symmetric pool
        (dp_nvlink.attach); the collectives then run over NVLink/NVSwitch."""
        reg = pool.regions[id(self)]
        if "param" in reg:
            v = pool.view(reg["param"], self.total)
            v.copy_(self.p_full)
            self.p_full = v
        if "grad" in reg:
            v = pool.view(reg["grad"], self.total)
            v.copy_(self.g_full)
            self.g_full = v
        self.nvl = pool

    # ------------------------------------------------------------------ values
    def views(self, flat: torch.Tensor) -> dict:
        return {n: flat[o:o + math.prod(s)].view(s) for n, (o, s) in self.layout.items()}

    def small_grads(self) -> dict:
        return {n: self.acc32[o:o + math.prod(s)].view(s) for n, (o, s) in
                self.small_layout.items()}

    def load(self, tensors: dict) -> None:
        """Fill parameters (and the fp32 master copy) from local tensors (any device)."""
        full = torch.zeros(self.total, dtype=torch.float32, device=self.device)
        for n, (o, s) in self.layout.items():
            t = tensors[n]
            if tuple(t.shape) != s:
                raise RuntimeError(f"{n}: expected {s}, got {tuple(t.shape)}")
            full[o:o + t.numel()] = t.reshape(-1).to(self.device, torch.float32)
        cast = full.to(self.dtype)
        if self.zero == 3:
            self.p_shard.copy_(cast[self.lo:self.lo + self.shard])
        else:
            self.p_full.copy_(cast)
        self._init_master(cast.float())

    def _init_master(self, full32: torch.Tensor) -> None:
        owned = full32 if self.zero == 0 else full32[self.lo:self.lo + self.shard]
        self.master = owned.clone()
        self.m = torch.zeros_like(owned)
        self.v = torch.zeros_like(owned)

    def _await_update(self) -> None:
        if self.ready_event is not None:
            torch.cuda.current_stream().wait_event(self.ready_event)
            self.ready_event = None

    def materialize(self) -> torch.Tensor:
        """Full flat parameters (z3: all-gather into a transient buffer, maybe prefetched)."""
        self._await_update()
        if self._param_epoch is not None:  # peers' fused AdamW + broadcast of their shards
            self.nvl.wait_params(self._param_epoch)
            self._param_epoch = None
        if self._param_ag is not None:  # post-step param all-gather still in flight
            self._param_ag[0].wait()
            self._param_ag = None
        if self.zero < 3:
            return self.p_full
        if self._gathered is None:
            self.prefetch()
        if self._gather_work is not None:
            self._gather_work.wait()
            self._gather_work = None
        return self._gathered

    def prefetch(self) -> None:
        """z3: start the parameter all-gather for the next use on the dp NCCL stream."""
        if self.zero < 3 or self._gathered is not None:
            return
        self._await_update()
        out = torch.empty(self.total, dtype=self.dtype, device=self.device)
        self._gather_work = _async(dist.all_gather_into_tensor, out, self.p_shard,
                                   group=self.dp.group)
        self._gathered = out

    def release(self) -> None:
        self._gathered = None
        self._gather_work = None

    # ------------------------------------------------------------------ grads
    def grad_target(self) -> torch.Tensor:
        self._await_update()
        if self.zero >= 2:
            if self.nvl is not None:
                self._slot, v = self.nvl.grad_slot(self.total)
                return v
            return torch.zeros(self.total, dtype=self.grad_dtype, device=self.device)
        return self.g_full

    def finish_microbatch(self, target: torch.Tensor, tp_partial=(), tp_group=None) -> None:
        """Fold the fp32 small-entry grads in; launch this layer's gradient collective
        asynchronously so it overlaps the backward of the layers below:
        z>=2 reduce-scatter into the shard accumulator every microbatch; z0/z1 the dp
        all-reduce / reduce-scatter after the last microbatch (DDP-style)."""
        sg = self.small_grads()
        for n in tp_partial:
            if n in sg:
                comm.all_reduce(sg[n], tp_group)
        views = self.views(target)
        for n, g in sg.items():
            K.axpby(g, views[n], 1.0, 1.0)
        self.acc32.zero_()
        if self.zero >= 2:
            comm.all_reduce(target, self.extra)
            if SKIP_DP_SYNC:
                self._slot = None
                return
            if self.nvl is not None:
                self.pending.append((self.nvl.reduce_scatter_slot(self, self._slot), None, ()))
                self._slot = None
                return
            part = torch.empty(self.shard, dtype=self.grad_dtype, device=self.device)
            work = _async(dist.reduce_scatter_tensor, part, target, group=self.dp.group)
            self.pending.append((work, lambda part=part: K.axpby(part, self.g_shard, 1.0, 1.0),
                                 (target, part)))
            _track(self)
        elif self.last_window:
            self._launch_sync()

    def _launch_sync(self) -> None:
        if self._synced:
            return
        self._synced = True
        if SKIP_DP_SYNC:
            if self.zero < 2:
                comm.all_reduce(self.g_full, self.extra)
            self._owned_grad = (self.g_full if self.zero == 0 else self.g_shard if
                                self.zero >= 2 else self.g_full[self.lo:self.lo + self.shard])
            return
        if self.zero < 2:
            comm.all_reduce(self.g_full, self.extra)
        if self.zero == 0:
            self._owned_grad = self.g_full
            if self.nvl is not None:
                self.pending.append((self.nvl.all_reduce_grad(self), None, ()))
            elif self.ndp > 1:
                self.pending.append((_async(dist.all_reduce, self.g_full, group=self.dp.group),
                                     None, ()))
        elif self.zero == 1:
            out = torch.empty(self.shard, dtype=self.grad_dtype, device=self.device)
            self._owned_grad = out
            if self.nvl is not None:
                self.pending.append((self.nvl.reduce_scatter_grad(self, out), None, (out,)))
                return
            self.pending.append((_async(dist.reduce_scatter_tensor, out, self.g_full,
                                        group=self.dp.group), None, (out,)))
        else:
            self._owned_grad = self.g_shard

    def drain(self) -> None:
        """Wait for this store's in-flight collectives and apply their epilogues."""
        for work, fin, _keep in self.pending:
            work.wait()
            if fin is not None:
                fin()
        self.pending.clear()

    def sync(self) -> None:
        """End of the accumulation window: dp reduction of the gradients."""
        self.drain()
        self._launch_sync()
        self.drain()
        self.last_window = False

    def owned_grad(self) -> torch.Tensor:
        return self._owned_grad

    def zero_grads(self) -> None:
        self._synced = False
        if self.g_full is not None:
            self.g_full.zero_()
        if self.g_shard is not None:
            self.g_shard.zero_()
        self.acc32.zero_()
        self._owned_grad = None

    def full_grad(self) -> torch.Tensor:
        """(tests) full flat gradient after sync, gathered across dp shards if needed."""
        if self.zero == 0:
            return self.g_full
        return comm.all_gather(self._owned_grad.contiguous(), self.dp)

    # ------------------------------------------------------------------ optimizer
    def step(self, *, lr, beta1, beta2, eps, weight_decay, step, grad_scale=1.0) -> None:
        g = self._owned_grad
        if g is not None and self.zero == 1:
            # the z1 shard grad was allocated on the compute stream and is read here on the
            # optimizer side stream; zero_grads() drops the last reference right after this
            # call is queued, so tell the caching allocator not to hand the block back to
            # the compute stream before the update has consumed it
            g.record_stream(torch.cuda.current_stream())
        if self.zero == 3:
            out = self.p_shard
        elif self.zero == 0:
            out = self.p_full
        else:
            out = self.p_full[self.lo:self.lo + self.shard]
        if SKIP_DP_SYNC and self.zero in (1, 2):
            K.adamw(self.master, self.m, self.v, g, out, lr=lr, beta1=beta1, beta2=beta2,
                    eps=eps, weight_decay=weight_decay, step=step, grad_scale=grad_scale)
            return
        if self.nvl is not None and self.zero in (1, 2):
            # fused AdamW + parameter all-gather over NVSwitch (dp_nvlink.py)
            self._param_epoch = self.nvl.adamw_bcast(
                self, g, lr=lr, beta1=beta1, beta2=beta2, eps=eps, weight_decay=weight_decay,
                step=step, grad_scale=grad_scale)
            return
        K.adamw(self.master, self.m, self.v, g, out, lr=lr, beta1=beta1, beta2=beta2, eps=eps,
                weight_decay=weight_decay, step=step, grad_scale=grad_scale)
        if self.zero in (1, 2):
            # in-place all-gather (input == output + rank*count): no temporary, so nothing is
            # allocated on the optimizer stream's allocator pool
            self._param_ag = (_async(dist.all_gather_into_tensor, self.p_full, out,
                                     group=self.dp.group), None)

    def memory_bytes(self) -> dict:
        def nb(t):
            return 0 if t is None else t.numel() * t.element_size()
        return {"param": nb(self.p_full) + nb(getattr(self, "p_shard", None)),
                "grad": nb(self.g_full) + nb(self.g_shard),
                "optimizer": nb(self.master) + nb(self.m) + nb(self.v)}
