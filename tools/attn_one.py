#!/usr/bin/env python
"""Launch one attention fwd (+ bwd) at a given shape a few times (for ncu captures).

    python tools/attn_one.py [--shape 2x4096x32x128] [--bwd] [--iters 3]"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="2x4096x32x128")
    ap.add_argument("--bwd", action="store_true")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    from paper_2504_21411_b200 import kernels as K
    B, S, H, D = (int(x) for x in a.shape.split("x"))
    qkv = torch.randn(B, S, 3, H, D, device="cuda").bfloat16()
    q, k, v = qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]
    o = torch.empty(B, S, H, D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, H, S, device="cuda")
    do = torch.randn_like(o)
    d = torch.empty_like(qkv)
    for _ in range(a.iters):
        K.attn_fwd(q, k, v, o, lse, scale=1 / math.sqrt(D), causal=True)
        if a.bwd:
            K.attn_bwd(q, k, v, o, do, lse, d[:, :, 0], d[:, :, 1], d[:, :, 2],
                       scale=1 / math.sqrt(D), causal=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
