"""Rank layout and communicators for a HybridConfig.

Contiguous placement, exactly the reference's modelling assumption
(collectives.py:36-46, 80-89): pipeline stages are contiguous rank blocks of
``devices_per_stage``; inside a stage, TP groups are consecutive ranks (TP
innermost) and DP groups stride by tp.  ``local = rank % devices_per_stage``,
``tp_rank = local % tp``, ``dp_rank = local // tp``.

Pure index math lives in module-level functions (tested on CPU); ``Topology``
creates the torch.distributed groups (NCCL on B200, gloo in CPU tests) once, in the
same order on every rank.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch.distributed as dist


def stage_of_rank(rank: int, devices_per_stage: int) -> int:
    return rank // devices_per_stage


def tp_members(stage: int, dps: int, tp: int, dp_rank: int) -> list:
    base = stage * dps + dp_rank * tp
    return list(range(base, base + tp))


def dp_members(stage: int, dps: int, tp: int, tp_rank: int) -> list:
    return [stage * dps + d * tp + tp_rank for d in range(dps // tp)]


@dataclass
class GroupHandle:
    """A communicator view: ranks, my index, and the torch group (None if size 1)."""

    ranks: tuple
    index: int
    group: object = None

    @property
    def size(self) -> int:
        return len(self.ranks)


class Topology:
    def __init__(self, hc, rank: int | None = None, world: int | None = None):
        self.hc = hc
        self.dps = hc.devices_per_stage
        self.distributed = dist.is_available() and dist.is_initialized()
        self.rank = rank if rank is not None else (dist.get_rank() if self.distributed else 0)
        self.world = world if world is not None else (
            dist.get_world_size() if self.distributed else 1)
        if self.world != hc.world_size:
            raise RuntimeError(f"plan needs {hc.world_size} ranks, launched with {self.world}")
        self.stage = stage_of_rank(self.rank, self.dps)
        self.local = self.rank % self.dps
        self._tp: dict = {}
        self._dp: dict = {}
        self._stage_group = None
        self._build()

    # every rank creates every group in the same order (torch.distributed requirement)
    def _build(self) -> None:
        tps = sorted({s.tp for s in self.hc.layer_strategies})
        for tp in tps:
            for stage in range(self.hc.pp):
                for d in range(self.dps // tp):
                    ranks = tp_members(stage, self.dps, tp, d)
                    g = self._new_group(ranks)
                    if self.rank in ranks:
                        self._tp[tp] = GroupHandle(tuple(ranks), ranks.index(self.rank), g)
                for t in range(tp):
                    ranks = dp_members(stage, self.dps, tp, t)
                    g = self._new_group(ranks)
                    if self.rank in ranks:
                        self._dp[tp] = GroupHandle(tuple(ranks), ranks.index(self.rank), g)
        for stage in range(self.hc.pp):
            ranks = list(range(stage * self.dps, (stage + 1) * self.dps))
            g = self._new_group(ranks)
            if self.rank in ranks:
                self._stage_group = GroupHandle(tuple(ranks), ranks.index(self.rank), g)

    def _new_group(self, ranks):
        if len(ranks) == 1 or not self.distributed:
            return None
        if len(ranks) == self.world:
            return dist.group.WORLD
        return dist.new_group(ranks)

    def tp(self, tp: int) -> GroupHandle:
        return self._tp[tp]

    def dp(self, tp: int) -> GroupHandle:
        return self._dp[tp]

    @property
    def stage_group(self) -> GroupHandle:
        return self._stage_group

    def prev_stage_rank(self) -> int | None:
        return self.rank - self.dps if self.stage > 0 else None

    def next_stage_rank(self) -> int | None:
        return self.rank + self.dps if self.stage < self.hc.pp - 1 else None
