"""Data-parallel gradient / parameter collectives over NVLink + NVSwitch (no NCCL).

The cost model's dp_sync (costmodel.py:199-213) is z0: AR(dp, grads); z>=1: RS(dp, grads)
+ AG(dp, params).  With NCCL those are ring passes that stream every byte through each
GPU (g-1) times and keep 16-32 SMs busy for the duration, next to the backward GEMMs.
Here every bf16 ZeRO-0/1/2 store's flat buffers of one dp group live in a single symmetric
allocation (torch symmetric memory as the allocator: every rank's pool is mapped into all
peers and bound to an NVSwitch multicast object), and the data movement is ours
(csrc/dp_nvlink.cu):

* grad reduce-scatter: each rank pulls its own chunk summed over the group with
  ``multimem.ld_reduce`` (the switch does the adds, each byte crosses NVLink once) and
  accumulates it into its shard in the same pass (ZeRO-2 per-microbatch accumulation);
* grad all-reduce (z0): the same pull plus a ``multimem.st`` of the reduced chunk;
* param all-gather (z1/z2) fused into AdamW: each rank stores its updated bf16 shard once
  to the multicast address and the switch writes it into every rank's full buffer.

Ordering: the reductions run on a per-pool comm stream bracketed by flag barriers on
channel 0 (ready before the pull, done after it, so buffers can be reused); the parameter
broadcast raises a channel-1 flag on the optimizer stream and each store's next use waits
for it on the compute stream with a single-CTA kernel.  Epochs are monotonic per channel
and each channel is only ever advanced from one stream, in the same store order on every
rank.  Without multicast (or GALV_DP_NVLINK_MC=0) the same kernels use unicast peer
loads/stores.  GALV_DP_NVLINK=0 falls back to NCCL (params.py).
"""

from __future__ import annotations

import os

import torch

from .. import kernels as K

_FLAGS = 512                  # [ch0 flags: 64 x u32][ch1 flags: 64 x u32][pad]
# ZeRO-2 grad-target slots: one being written by the current layer's backward while the
# previous layer's is reduced on the comm stream (a 400 MB pull-reduce takes ~0.6 ms, a
# layer backward ~20 ms, so a third slot only costs memory)
RING = int(os.environ.get("GALV_DP_RING", "2"))
# CTAs of the pull-reduce kernels: B200, one 7B layer's gradients (405 MB) at N=2, alone
# (tools/nvlink_bench.py, profiles/r02/nvlink): 16 CTAs 184 GB/s busbw, 32 316, 64 321, NCCL
# 374; inside the step (profiler --overlap-out) the exposed dp sync fell from 60 / 48 ms
# (16 CTAs, N=2 / 4) to 30 / 25 ms with 48 CTAs (NCCL 32 / 45 ms)
MAX_CTAS = int(os.environ.get("GALV_DP_NVLINK_CTAS", "48"))


def enabled() -> bool:
    return os.environ.get("GALV_DP_NVLINK", "1") != "0"


def _eligible(store) -> bool:
    return (store.dp is not None and store.ndp > 1 and store.zero in (0, 1, 2)
            and store.dtype == torch.bfloat16 and store.grad_dtype == torch.bfloat16)


class _EventWork:
    """Work handle for ParamStore.pending: wait = make the current stream wait the event."""

    def __init__(self, ev):
        self.ev = ev

    def wait(self):
        torch.cuda.current_stream().wait_event(self.ev)


class DpPool:
    def __init__(self, group, stores, device):
        import torch.distributed._symmetric_memory as symm_mem
        self.g = group
        self.t, self.me = group.size, group.index
        self.device = device
        off = _FLAGS
        self.regions = {}
        ring_elems = 0
        for st in stores:
            reg = {}
            if st.zero in (1, 2):
                reg["param"] = off
                off += st.total * 2
            if st.zero in (0, 1):
                reg["grad"] = off
                off += st.total * 2
            else:
                ring_elems = max(ring_elems, st.total)
            self.regions[id(st)] = reg
        self.ring = []
        for _ in range(RING if ring_elems else 0):
            self.ring.append([off, None])       # [byte offset, release event]
            off += ring_elems * 2
        self.ring_elems = ring_elems
        self.nbytes = (off + 4095) // 4096 * 4096
        self.buf = symm_mem.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.buf[:_FLAGS].zero_()
        torch.cuda.synchronize()
        hdl = symm_mem.rendezvous(self.buf, group.group)
        self.ptrs = [int(p) for p in hdl.buffer_ptrs]
        mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
        self.mc = mc if os.environ.get("GALV_DP_NVLINK_MC", "1") != "0" else 0
        self.flag_ptrs = [torch.tensor([p + c * 256 for p in self.ptrs], dtype=torch.int64,
                                       device=device) for c in (0, 1)]
        self.my_flags = [self.ptrs[self.me] + c * 256 for c in (0, 1)]
        self._peer_cache = {}
        self.epoch = [0, 0]
        self.comm = torch.cuda.Stream(device=device)
        self.next_slot = 0
        torch.distributed.barrier(group=group.group)

    # ------------------------------------------------------------------ addressing
    def view(self, byte_off: int, n: int) -> torch.Tensor:
        return self.buf[byte_off:byte_off + 2 * n].view(torch.bfloat16)

    def peers(self, byte_off: int) -> torch.Tensor:
        """Device array of every rank's address of the region at byte_off."""
        t = self._peer_cache.get(byte_off)
        if t is None:
            t = torch.tensor([p + byte_off for p in self.ptrs], dtype=torch.int64,
                             device=self.device)
            self._peer_cache[byte_off] = t
        return t

    def _mc(self, byte_off: int, elem_off: int):
        return self.mc + byte_off + 2 * elem_off if self.mc else None

    # ------------------------------------------------------------------ sync primitives
    def _barrier(self, ch: int = 0) -> None:
        self.epoch[ch] += 1
        K.nvl_signal(self.flag_ptrs[ch], self.me, self.t, self.epoch[ch])
        K.nvl_wait(self.my_flags[ch], self.t, self.epoch[ch])

    def _reduce(self, byte_off, lo, n, *, out=None, accumulate=False, bcast=False):
        """On the comm stream, after the current stream's work: barrier, pull-reduce
        [lo, lo+n) of the region at byte_off, barrier.  Returns the completion event."""
        ready = torch.cuda.Event()
        ready.record()
        with torch.cuda.stream(self.comm):
            self.comm.wait_event(ready)
            self._barrier(0)
            if self.mc:
                K.dp_reduce(n=n, t=self.t, mc_src=self._mc(byte_off, lo), out=out,
                            accumulate=accumulate,
                            mc_dst=self._mc(byte_off, lo) if bcast else None,
                            max_ctas=MAX_CTAS)
            else:
                p = self.peers(byte_off)
                K.dp_reduce(n=n, t=self.t, peer_src=p, offset=lo, out=out,
                            accumulate=accumulate, peer_dst=p if bcast else None,
                            max_ctas=MAX_CTAS)
            self._barrier(0)
            done = torch.cuda.Event()
            done.record()
        return done

    # ------------------------------------------------------------------ store operations
    def grad_slot(self, n: int) -> tuple:
        """Next ZeRO-2 grad-target slot (zeroed on the current stream once free)."""
        slot = self.ring[self.next_slot]
        self.next_slot = (self.next_slot + 1) % len(self.ring)
        if slot[1] is not None:
            torch.cuda.current_stream().wait_event(slot[1])
            slot[1] = None
        v = self.view(slot[0], n)
        v.zero_()
        return slot, v

    def reduce_scatter_slot(self, store, slot) -> _EventWork:
        done = self._reduce(slot[0], store.lo, store.shard, out=store.g_shard, accumulate=True)
        slot[1] = done
        return _EventWork(done)

    def reduce_scatter_grad(self, store, out) -> _EventWork:
        return _EventWork(self._reduce(self.regions[id(store)]["grad"], store.lo, store.shard,
                                       out=out))

    def all_reduce_grad(self, store) -> _EventWork:
        """z0: each rank reduces its dp chunk and stores it to all ranks (two-shot)."""
        return _EventWork(self._reduce(self.regions[id(store)]["grad"], store.lo, store.shard,
                                       bcast=True))

    def adamw_bcast(self, store, g, **hyper) -> int:
        """Fused AdamW + parameter all-gather on the current (optimizer) stream; returns the
        channel-1 epoch the next use of this store waits for."""
        off = self.regions[id(store)]["param"]
        if self.mc:
            K.adamw_bcast(store.master, store.m, store.v, g, t=self.t, offset=store.lo,
                          mc_dst=self._mc(off, store.lo), **hyper)
        else:
            K.adamw_bcast(store.master, store.m, store.v, g, t=self.t, offset=store.lo,
                          peer_dst=self.peers(off), **hyper)
        self.epoch[1] += 1
        K.nvl_signal(self.flag_ptrs[1], self.me, self.t, self.epoch[1])
        return self.epoch[1]

    def wait_params(self, epoch: int) -> None:
        K.nvl_wait(self.my_flags[1], self.t, epoch)


def attach(stores, device) -> list:
    """Move every eligible store's flat buffers into one symmetric pool per dp group.
    Collective over each dp group (call on every rank, same store order)."""
    if not enabled() or torch.device(device).type != "cuda":
        return []
    groups = {}
    for st in stores:
        if _eligible(st):
            groups.setdefault(tuple(st.dp.ranks), (st.dp, []))[1].append(st)
    pools = []
    for _, (grp, sts) in groups.items():
        pool = DpPool(grp, sts, device)
        for st in sts:
            st.attach_nvlink(pool)
        pools.append(pool)
    return pools
