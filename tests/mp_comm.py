"""torchrun worker: the C-ABI NCCL layer (galv_comm_* / galv_all_reduce ...) vs torch.distributed.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mp_comm.py
"""

import os
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2504_21411_b200 import kernels as K  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = [K.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = K.comm_init(uid[0], world, rank)
    ok = True
    g = torch.Generator(device="cuda").manual_seed(7 + rank)
    for dtype in (torch.float32, torch.bfloat16):
        x = torch.randn(4096 * world, device="cuda", generator=g).to(dtype)
        ref = x.clone()
        dist.all_reduce(ref)
        got = K.comm_all_reduce(comm, x.clone())
        ok &= torch.equal(got, ref)
        rs = torch.empty(4096, device="cuda", dtype=dtype)
        K.comm_reduce_scatter(comm, x, rs)
        rref = torch.empty_like(rs)
        dist.reduce_scatter_tensor(rref, x)
        ok &= torch.equal(rs, rref)
        ag = torch.empty(4096 * world * world, device="cuda", dtype=dtype)
        K.comm_all_gather(comm, x, ag)
        aref = torch.empty_like(ag)
        dist.all_gather_into_tensor(aref, x)
        ok &= torch.equal(ag, aref)
    # ring exchange with grouped send/recv (pipeline boundary pattern)
    s = torch.full((1024,), float(rank), device="cuda")
    r = torch.empty_like(s)
    K.comm_sendrecv(comm, s, (rank + 1) % world, r, (rank - 1) % world)
    torch.cuda.synchronize()
    ok &= bool((r == float((rank - 1) % world)).all())
    # split into even/odd ranks and all-reduce inside the halves
    sub = K.comm_split(comm, rank % 2, rank)
    y = torch.ones(256, device="cuda")
    K.comm_all_reduce(sub, y)
    torch.cuda.synchronize()
    ok &= bool((y == float(len(range(rank % 2, world, 2)))).all())
    K.comm_destroy(sub)
    K.comm_destroy(comm)
    print(f"[rank {rank}] comm: {'PASS' if ok else 'FAIL'}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
