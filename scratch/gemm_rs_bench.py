import os, sys, torch, torch.distributed as dist
sys.path.insert(0, '.')
from paper_2504_21411_b200 import kernels as K
from paper_2504_21411_b200.runtime.nvlink import PeerBuffers
from paper_2504_21411_b200.runtime.topology import GroupHandle
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
t = dist.get_world_size(); me = dist.get_rank()
g = GroupHandle(tuple(range(t)), me, dist.group.WORLD)
def timeit(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); dist.barrier()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b)/it], device='cuda'); dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return ms.item()
for (M, N, Kd) in [(16384, 4096, 11008 // t), (16384, 4096, 4096 // t), (32768, 5120, 13824 // t)]:
    torch.manual_seed(me)
    a = torch.randn(M, Kd, device='cuda').bfloat16(); w = torch.randn(N, Kd, device='cuda').bfloat16()
    pb = PeerBuffers(g, M * N * 2, 'cuda')
    out = torch.empty(M // t, N, device='cuda', dtype=torch.bfloat16)
    def nccl():
        y = K.gemm(a, w, trans_b=True); dist.reduce_scatter_tensor(out, y)
    def fused():
        return pb.gemm_rs(a, w, trans_b=True)
    def gemm_only():
        K.gemm(a, w, trans_b=True)
    r1 = fused(); y = K.gemm(a, w, trans_b=True); ref = torch.empty_like(out); dist.reduce_scatter_tensor(ref, y)
    err = ((r1.float()-ref.float()).norm()/ref.float().norm()).item()
    tg, tn, tf = timeit(gemm_only), timeit(nccl), timeit(fused)
    if me == 0:
        print(f"t={t} M{M} N{N} K{Kd}: gemm {tg:.3f} ms | gemm+NCCL RS {tn:.3f} ms | fused NVLink {tf:.3f} ms | err {err:.1e}", flush=True)
dist.destroy_process_group()
