#!/usr/bin/env python
"""NVLink / NVSwitch collective kernels vs NCCL on the same box (torchrun, N ranks).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nvlink_bench.py [--out F]

* dp reduce-scatter (the ZeRO-2 gradient sync, costmodel.py:199-213): galv_dp_reduce
  pulling each rank's chunk through NVSwitch multimem.ld_reduce, vs
  dist.reduce_scatter_tensor, on one Llama-2-7B layer's bf16 gradients (202.4 M).
  busbw = (t-1)/t * bytes / time (the ring-pass convention of collectives.py:49-57).
* tp GEMM + reduce-scatter (Megatron-SP row-parallel GEMM, costmodel.py:108-112):
  galv_gemm_rs (epilogue stores rows into the owning rank's NVLink receive slot) + the
  slot reduce, vs galv GEMM followed by dist.reduce_scatter_tensor, at the Llama-2-13B
  down-projection shape of config C5 (tokens 32768, K = 13824/t, N = 5120).
Device time with CUDA events on the launching stream, max over ranks, median of 10.
"""

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, iters=10, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    out = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out.append(t.item() * 1e3)
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t, me = dist.get_world_size(), dist.get_rank()
    from paper_2504_21411_b200 import kernels as K
    from paper_2504_21411_b200.runtime import nvlink
    from paper_2504_21411_b200.runtime.topology import GroupHandle
    import torch.distributed._symmetric_memory as symm_mem
    res = {"world": t}
    # ---- dp reduce-scatter
    n = 202_383_360 // (t * 64) * (t * 64)
    buf = symm_mem.empty(n * 2, dtype=torch.uint8, device="cuda")
    hdl = symm_mem.rendezvous(buf, dist.group.WORLD)
    mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
    buf.view(torch.bfloat16).normal_()
    shard = n // t
    out = torch.empty(shard, dtype=torch.bfloat16, device="cuda")
    peers = torch.tensor([int(p) for p in hdl.buffer_ptrs], dtype=torch.int64, device="cuda")
    nbytes = n * 2
    if mc:
        for ctas in (16, 32, 64, 148):
            us = timed(lambda: K.dp_reduce(n=shard, t=t, mc_src=mc + me * shard * 2, out=out,
                                           max_ctas=ctas))
            res[f"galv_dp_reduce_multimem_ctas{ctas}"] = {
                "us": us, "busbw_GBps": (t - 1) / t * nbytes / us / 1e3}
    us = timed(lambda: K.dp_reduce(n=shard, t=t, peer_src=peers, offset=me * shard, out=out,
                                   max_ctas=16))
    res["galv_dp_reduce_unicast"] = {"us": us, "busbw_GBps": (t - 1) / t * nbytes / us / 1e3}
    src = buf.view(torch.bfloat16)
    us = timed(lambda: dist.reduce_scatter_tensor(out, src))
    res["nccl_reduce_scatter"] = {"us": us, "busbw_GBps": (t - 1) / t * nbytes / us / 1e3}
    # ---- tp GEMM + reduce-scatter (C5 down projection)
    T, F, N = 32768, 13824 // t, 5120
    a = torch.randn(T, F, device="cuda", dtype=torch.bfloat16) * 0.1
    w = torch.randn(N, F, device="cuda", dtype=torch.bfloat16) * 0.1
    grp = GroupHandle(tuple(range(t)), me, dist.group.WORLD)
    pb = nvlink.PeerBuffers(grp, T * N * 2, torch.device("cuda", local))
    us_f = timed(lambda: pb.gemm_rs(a, w, trans_b=True))
    part = torch.empty(T // t, N, device="cuda", dtype=torch.bfloat16)

    def unfused():
        y = K.gemm(a, w, trans_b=True)
        dist.reduce_scatter_tensor(part, y)
    us_u = timed(unfused)
    us_g = timed(lambda: K.gemm(a, w, trans_b=True))
    flops = 2.0 * T * F * N
    res["gemm_rs_c5_down"] = {"shape": [T, N, F], "fused_us": us_f, "gemm_plus_nccl_rs_us": us_u,
                              "gemm_alone_us": us_g, "fused_tflops": flops / us_f / 1e6,
                              "exposed_comm_fused_us": us_f - us_g,
                              "exposed_comm_nccl_us": us_u - us_g,
                              "rs_bytes_per_rank": (t - 1) / t * T * N * 2}
    if me == 0:
        print(json.dumps(res), flush=True)
        if args.out:
            with open(args.out, "a") as fh:
                fh.write(json.dumps(res) + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
