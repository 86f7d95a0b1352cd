"""clock64 timeline of the dK/dV kernel's CTA (0, 0) (key block 0: 32 query steps at S=4096).

Needs a library built with -DGALV_ATTN_TRACE (TRACE points compiled in), e.g.
    for f in paper_2504_21411_b200/csrc/*.cu; do nvcc -gencode arch=compute_100a,code=sm_100a \
        -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include -DGALV_ATTN_TRACE \
        -c $f -o /tmp/tr/$(basename $f .cu).o; done
    nvcc -shared -gencode arch=compute_100a,code=sm_100a -o /tmp/libgalv_trace.so /tmp/tr/*.o -lcudart -ldl
    python tools/attn_bwd_trace.py /tmp/libgalv_trace.so
Columns: MMA-warp issue points (m:) and math warp 4 (s:) per query step, SM cycles."""
import sys, math, ctypes, torch, numpy as np
sys.path.insert(0, '.')
from paper_2504_21411_b200 import kernels as K
K._lib = K.load_library(sys.argv[1] if len(sys.argv) > 1 else 'scratch/libgalv_trace.so')
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
b = buf.astype(np.int64)
base = 4096
t0 = b[base + 16*64 + 3]
t = b[base: base + 32*16].reshape(32, 16) - t0
print("start->kv_full seen", b[base+16*64+2]-t0, " mm_done seen", b[base+16*64]-t0, " epilogue end", b[base+16*64+1]-t0)
cols = [(0,"m:pwait"),(1,"m:dV"),(2,"m:S+1"),(3,"m:dK"),(4,"m:dP+1"),(8,"s:Sseen"),(9,"s:Pdone"),(10,"s:Parr"),(11,"s:dPseen"),(12,"s:dSarr")]
print("it " + " ".join(f"{n:>9}" for _,n in cols))
for i in range(32):
    print(f"{i:2d} " + " ".join(f"{t[i,c]:9d}" for c,_ in cols))
r = slice(3, 29)
print("period (dV issue)", np.diff(t[:,1])[r].mean())
print("phase1 S seen -> P arrive", (t[:,10]-t[:,8])[r].mean(), " exp part", (t[:,9]-t[:,8])[r].mean())
print("phase1 S seen -> S loaded", (t[:,13]-t[:,8])[r].mean(), " phase2 dP seen -> dP half loaded", (t[:,14]-t[:,11])[r].mean())
print("phase2 dP seen -> dS arrive", (t[:,12]-t[:,11])[r].mean())
print("P arrive -> dV issue", (t[:,1]-t[:,10])[r].mean(), " dS arrive -> dK issue", (t[:,3]-t[:,12])[r].mean())
print("S(it+1) issue -> S seen(it+1)", (t[1:,8]-t[:-1,2])[r].mean(), " dP(it+1) issue -> dP seen", (t[1:,11]-t[:-1,4])[r].mean())
print("waits: s_full wait start (after dS arr) -> S seen", (t[1:,8]-t[:-1,12])[r].mean(), " P arr -> dP seen", (t[:,11]-t[:,10])[r].mean())
