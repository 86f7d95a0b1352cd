"""Inter-layer strategy transition: one row-gather pack kernel, ONE all-to-all, one
row-scatter unpack kernel (the realization of costmodel.transition_time,
reference costmodel.py:179-196, which bounds it by an all-gather of the boundary
tensor over the stage group).

A layout is (tp, dp, sp) on a stage of n = tp*dp ranks.  For a microbatch of T
tokens (token-major [b, s]), rank ``local = dp_rank*tp + tp_rank`` holds the
contiguous token range
    rep = T/dp, lo = dp_rank*rep (+ tp_rank*rep/tp if sp), length rep (rep/tp if sp).
Replicas (sp=False, tp>1) hold identical rows and, by construction of the layers'
backward, identical full gradients, so the backward of a transition is the
transition in the opposite direction.  Only rows a rank lacks move; a transition that
merely shrinks a rank's range (e.g. sp=False -> sp=True at equal dp) moves nothing
over the network.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Layout:
    tp: int
    dp: int
    sp: bool

    @classmethod
    def of(cls, strategy) -> "Layout":
        return cls(strategy.tp, strategy.dp, bool(strategy.sp and strategy.tp > 1))

    def token_range(self, local: int, T: int) -> tuple:
        rep = T // self.dp
        d, t = divmod(local, self.tp)
        if self.sp:
            chunk = rep // self.tp
            lo = d * rep + t * chunk
            return lo, lo + chunk
        return d * rep, (d + 1) * rep

    def holders(self, token: int, T: int) -> list:
        """Local ranks holding ``token``."""
        rep = T // self.dp
        d = token // rep
        if self.sp:
            t = (token - d * rep) // (rep // self.tp)
            return [d * self.tp + t]
        return [d * self.tp + t for t in range(self.tp)]


@dataclass
class TransitionPlan:
    """Per-rank send/recv schedule for one direction of one transition."""

    send_rows: list        # per rank: list (over destinations) of (lo, hi) local row ranges
    recv_rows: list        # per rank: list (over sources) of (lo, hi) dst-local row ranges
    moves_data: bool

    def for_rank(self, local: int):
        return self.send_rows[local], self.recv_rows[local]


def plan_transition(src: Layout, dst: Layout, T: int) -> TransitionPlan:
    """Which rows every rank sends to / receives from every other rank."""
    n = src.tp * src.dp
    assert dst.tp * dst.dp == n, "transition within one stage group"
    # pieces: for each dst rank, split its needed range at src chunk boundaries
    src_cuts = sorted({src.token_range(i, T)[k] for i in range(n) for k in (0, 1)})
    send = [[(0, 0)] * n for _ in range(n)]   # send[src_rank][dst_rank] = src-local range
    recv = [[(0, 0)] * n for _ in range(n)]   # recv[dst_rank][src_rank] = dst-local range
    moves = False
    for j in range(n):
        dlo, dhi = dst.token_range(j, T)
        cuts = [c for c in src_cuts if dlo < c < dhi]
        bounds = [dlo] + cuts + [dhi]
        for a, b in zip(bounds[:-1], bounds[1:]):
            if a == b:
                continue
            hs = src.holders(a, T)
            owner = j if j in hs else hs[j % len(hs)]
            slo, _ = src.token_range(owner, T)
            prev = send[owner][j]
            # pieces from one owner to one destination are contiguous by construction
            if prev == (0, 0):
                send[owner][j] = (a - slo, b - slo)
                recv[j][owner] = (a - dlo, b - dlo)
            else:
                send[owner][j] = (prev[0], b - slo)
                recv[j][owner] = (recv[j][owner][0], b - dlo)
            if owner != j:
                moves = True
    return TransitionPlan(send_rows=send, recv_rows=recv, moves_data=moves)


_PLAN_CACHE: dict = {}


def cached_plan(src: Layout, dst: Layout, T: int) -> TransitionPlan:
    key = (src, dst, T)
    if key not in _PLAN_CACHE:
        _PLAN_CACHE[key] = plan_transition(src, dst, T)
    return _PLAN_CACHE[key]


def index_tensors(plan: TransitionPlan, local: int, device):
    """(send_idx, send_splits, recv_idx, recv_splits) for the pack / unpack kernels."""
    send, recv = plan.for_rank(local)
    sidx = [torch.arange(lo, hi) for lo, hi in send]
    ridx = [torch.arange(lo, hi) for lo, hi in recv]
    s_splits = [hi - lo for lo, hi in send]
    r_splits = [hi - lo for lo, hi in recv]
    cat = lambda xs: torch.cat(xs) if xs else torch.zeros(0, dtype=torch.int64)
    return (cat(sidx).to(device), s_splits, cat(ridx).to(device), r_splits)


class Resharder:
    """Applies transitions on a stage group with galv pack/unpack kernels + NCCL all-to-all."""

    def __init__(self, stage_group, local: int, device):
        self.g, self.local, self.device = stage_group, local, device
        self._idx: dict = {}

    def __call__(self, x: torch.Tensor, src: Layout, dst: Layout, T: int) -> torch.Tensor:
        if src == dst:
            return x
        from .. import kernels as K
        from . import comm
        plan = cached_plan(src, dst, T)
        key = (src, dst, T)
        if key not in self._idx:
            self._idx[key] = index_tensors(plan, self.local, self.device)
        sidx, ss, ridx, rs = self._idx[key]
        lo, hi = dst.token_range(self.local, T)
        out = torch.empty(hi - lo, x.shape[1], dtype=x.dtype, device=x.device)
        if not plan.moves_data:
            # every needed row is local: one gather kernel, no collective
            s_lo = sum(ss[:self.local])
            K.gather_rows(x, sidx[s_lo:s_lo + ss[self.local]], out)
            return out
        send = torch.empty(sum(ss), x.shape[1], dtype=x.dtype, device=x.device)
        if send.shape[0]:
            K.gather_rows(x, sidx, send)
        recv = torch.empty(sum(rs), x.shape[1], dtype=x.dtype, device=x.device)
        comm.all_to_all(recv, send, rs, ss, self.g)
        if recv.shape[0]:
            K.scatter_rows(recv, ridx, out)
        return out
