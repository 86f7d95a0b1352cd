"""clock64 timeline of bwd dq CTA (0,0) from the GALV_ATTN_TRACE build (scratch/libgalv_trace.so)."""
import sys, math, ctypes, torch, numpy as np
sys.path.insert(0, '.')
from paper_2504_21411_b200 import kernels as K
K._lib = K.load_library('scratch/libgalv_trace.so')
lib = K._lib
B,S,H,D = 2,4096,32,128
qkv = torch.randn(B*S, 3*H*D, device='cuda').bfloat16()
mk = lambda j: qkv.as_strided((B,S,H,D),(S*3*H*D,3*H*D,D,1), j*H*D)
q,k,v = mk(0),mk(1),mk(2)
o = torch.empty(B,S,H,D,device='cuda',dtype=torch.bfloat16); lse=torch.empty(B,H,S,device='cuda')
K.attn_fwd(q,k,v,o,lse,scale=1/math.sqrt(D),causal=True)
dqkv = torch.empty_like(qkv)
dq,dk,dv = [dqkv.as_strided((B,S,H,D),(S*3*H*D,3*H*D,D,1), j*H*D) for j in range(3)]
do = torch.randn_like(o)
ws = torch.empty(K.attn_bwd_workspace_bytes(B,S,H,D,torch.bfloat16), dtype=torch.uint8, device="cuda")
for _ in range(3):
    K.attn_bwd(q,k,v,o,do,lse,dq,dk,dv,scale=1/math.sqrt(D),causal=True,workspace=ws)
torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64)
lib.galv_attn_trace_read.argtypes = [ctypes.c_void_p]
assert lib.galv_attn_trace_read(buf.ctypes.data) == 0
t = buf[:32*8].reshape(32, 8).astype(np.int64)
t = t - t[0, 0]
names = ["mma:loop", "mma:S", "mma:dP", "mma:dQ", "sm:st_full", "sm:ld", "sm:comp", "sm:ds_arr"]
print("it " + " ".join(f"{n:>10}" for n in names))
for i in range(32):
    print(f"{i:2d} " + " ".join(f"{x:10d}" for x in t[i]))
d = np.diff(t[:, 1])
print("S issue interval mean", d[2:].mean())
print("softmax: wait->ld", (t[:,5]-t[:,4])[2:].mean(), " ld->comp", (t[:,6]-t[:,5])[2:].mean(), " comp->arr", (t[:,7]-t[:,6])[2:].mean())
print("dQ issue - ds_arr", (t[:,3]-t[:,7])[2:].mean())
print("S issue - dQ(it-2) issue", (t[2:,1]-t[:-2,3])[2:].mean())
print("st_full seen - dP issue", (t[:,4]-t[:,2])[2:].mean())
print("==== dkdv CTA (0,0): 64 x 64-query steps")
t = buf[4096:4096 + 64*8].reshape(64, 8).astype(np.int64)
t = t - t[0, 0]
names = ["mma:loop", "mma:S", "mma:qful", "mma:grad", "sm:st_full", "sm:ld", "sm:comp", "sm:p_arr"]
print("it " + " ".join(f"{n:>10}" for n in names))
for i in list(range(0, 12)) + list(range(58, 64)):
    print(f"{i:2d} " + " ".join(f"{x:10d}" for x in t[i]))
print("S issue interval mean", np.diff(t[:, 1])[4:-4].mean())
print("loop->qfull", (t[:,2]-t[:,0])[4:-4].mean(), "qfull->S", (t[:,1]-t[:,2])[4:-4].mean())
print("softmax: wait->ld", (t[:,5]-t[:,4])[4:-4].mean(), " ld->comp", (t[:,6]-t[:,5])[4:-4].mean(), " comp->arr", (t[:,7]-t[:,6])[4:-4].mean())
print("grad issue - p_arr", (t[:,3]-t[:,7])[4:-4].mean())
print("st_full seen - S issue", (t[:,4]-t[:,1])[4:-4].mean())
print("==== fwd CTA (0,0) (heaviest q block): 32 KV blocks")
K.attn_fwd(q,k,v,o,lse,scale=1/math.sqrt(D),causal=True)
torch.cuda.synchronize()
assert lib.galv_attn_trace_read(buf.ctypes.data) == 0
t = buf[6144:6144 + 32*8].reshape(32, 8).astype(np.int64)
t = t - t[0, 6]
names = ["mma:S", "mma:PV", "sm:s_full", "sm:ld", "sm:exp", "sm:p_arr", "mma:top", "mma:kful"]
print("j  " + " ".join(f"{n:>10}" for n in names))
for i in range(32):
    print(f"{i:2d} " + " ".join(f"{x:10d}" for x in t[i]))
m = slice(3, 29)
print("block interval (S issue)", np.diff(t[:, 0])[m].mean())
print("s_full seen - S issue", (t[:,2]-t[:,0])[m].mean(), " ld", (t[:,3]-t[:,2])[m].mean(), " exp", (t[:,4]-t[:,3])[m].mean(), " exp->arr", (t[:,5]-t[:,4])[m].mean())
print("PV issue - p_arr", (t[:,1]-t[:,5])[m].mean())
print("top->kfull", (t[:,7]-t[:,6])[m].mean(), " kfull->S(s_empty)", (t[:,0]-t[:,7])[m].mean())
