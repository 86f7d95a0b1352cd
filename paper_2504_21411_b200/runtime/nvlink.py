"""Symmetric NVLink buffers for the tensor-parallel group (the fused GEMM + reduce-scatter).

torch.distributed._symmetric_memory is used only as the allocator / handle exchange
(plumbing): it maps every rank's buffer into every peer so that galv kernels can store to
peer addresses.  The data movement is ours: the row-parallel GEMM epilogue writes each
output row into the owning rank's receive slot (kernels.gemm_rs), and
galv_tp_signal_reduce raises a flag on every peer, waits for all, and sums the slots.

Layout of one rank's symmetric allocation: [flags: 256 B][recv 0][recv 1][gather 0][gather 1];
consecutive calls alternate buffers (call parity) so a fast rank can never overwrite data a
slow rank is still reducing (a rank can run at most one call ahead of any peer).  Flag epochs
increase monotonically (one per signal round).

* ``gemm_rs``: Megatron-SP row-parallel GEMM -> this rank's reduced token chunk.
* ``gemm_ar``: non-SP row-parallel GEMM -> full all-reduced output: the fused GEMM +
  reduce-scatter above, then every rank stores its reduced chunk straight into all peers'
  gather buffers (NVLink peer stores) and signals -- an all-reduce with no NCCL call.
"""

from __future__ import annotations

import os

import torch

from .. import kernels as K

_FLAG_BYTES = 256
_CACHE: dict = {}


def enabled() -> bool:
    """Fused GEMM + reduce-scatter over NVLink for Megatron-SP layers (default on: measured
    at or above NCCL, e.g. Llama-2-13B@32K tp2 24.5k vs 24.4k tok/s)."""
    return os.environ.get("GALV_TP_NVLINK", "1") != "0"


def allreduce_enabled() -> bool:
    """The NVLink all-reduce (fused GEMM-RS + peer-store all-gather) for non-SP TP layers is
    opt-in: NCCL's all-reduce (NVLS on NVSwitch) measured 2.5 % faster end to end on the
    GPT-1.3B alternating-strategy config."""
    return os.environ.get("GALV_TP_NVLINK_AR", "0") == "1"


class PeerBuffers:
    def __init__(self, group, region_bytes: int, device):
        import torch.distributed._symmetric_memory as symm_mem
        self.g = group
        self.t, self.me = group.size, group.index
        self.region = (region_bytes + 255) // 256 * 256
        self.buf = symm_mem.empty(_FLAG_BYTES + 4 * self.region, dtype=torch.uint8, device=device)
        self.buf[:_FLAG_BYTES].zero_()
        torch.cuda.synchronize()
        hdl = symm_mem.rendezvous(self.buf, group.group)
        ptrs = [int(p) for p in hdl.buffer_ptrs]
        self.flag_ptrs = torch.tensor(ptrs, dtype=torch.int64, device=device)
        self.data_ptrs = [torch.tensor([p + _FLAG_BYTES + k * self.region for p in ptrs],
                                       dtype=torch.int64, device=device) for k in (0, 1)]
        self.gather_ptrs = [torch.tensor([p + _FLAG_BYTES + (2 + k) * self.region for p in ptrs],
                                         dtype=torch.int64, device=device) for k in (0, 1)]
        self.epoch = 0
        self.calls = 0
        torch.distributed.barrier(group=group.group)

    def _region(self, idx: int, nbytes: int):
        off = _FLAG_BYTES + idx * self.region
        return self.buf[off:off + nbytes]

    def gemm_rs(self, a, b, *, trans_b: bool, out_dtype=torch.bfloat16):
        """op(a) @ op(b) summed over the tp group, this rank's row chunk: [rows/t, N]."""
        M = a.shape[0]
        N = b.shape[0] if trans_b else b.shape[1]
        rows = M // self.t
        if M % self.t or M * N * 2 > self.region:
            raise RuntimeError("gemm_rs: shape does not fit the symmetric buffer")
        self.calls += 1
        k = self.calls & 1
        self.epoch += 1
        K.gemm_rs(a, b, self.data_ptrs[k], rows, self.me, trans_b=trans_b, ldc=N)
        recv = self._region(k, M * N * 2).view(torch.bfloat16)
        out = torch.empty(rows, N, dtype=out_dtype, device=a.device)
        K.tp_signal_reduce(self.flag_ptrs, self.me, self.t, self.epoch, recv, out)
        return out

    def gemm_ar(self, a, b, *, trans_b: bool):
        """op(a) @ op(b) all-reduced over the tp group: [M, N] on every rank."""
        chunk = self.gemm_rs(a, b, trans_b=trans_b)
        k = self.calls & 1
        M, N = a.shape[0], chunk.shape[1]
        self.epoch += 1
        K.tp_allgather(chunk, self.gather_ptrs[k], self.flag_ptrs, self.me, self.t, self.epoch)
        return self._region(2 + k, M * N * 2).view(torch.bfloat16).view(M, N).clone()


def symmetric_bytes() -> int:
    """Bytes of the live tp peer-buffer allocations (symmetric memory: outside the caching
    allocator, so torch.cuda.max_memory_allocated does not see them)."""
    return sum(pb.buf.numel() * pb.buf.element_size() for pb in _CACHE.values())


def peer_buffers(group, region_bytes: int, device) -> PeerBuffers:
    """Shared per tp group; grows (collectively, in layer-construction order) if needed."""
    key = tuple(group.ranks)
    pb = _CACHE.get(key)
    if pb is None or pb.region < region_bytes:
        pb = PeerBuffers(group, region_bytes, device)
        _CACHE[key] = pb
    return pb
