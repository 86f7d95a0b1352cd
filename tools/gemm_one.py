#!/usr/bin/env python
"""Launch the step's largest GEMM a few times (for ncu --set full captures): the Llama-2-7B
gate|up projection with the SwiGLU epilogue at microbatch 2 (8192 x 22016 x 4096).

    python tools/gemm_one.py [--iters 4] [--shape M,F,K]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--shape", default="8192,11008,4096")
    a = ap.parse_args()
    from paper_2504_21411_b200 import kernels as K
    M, F, Kd = (int(x) for x in a.shape.split(","))
    x = torch.randn(M, Kd, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(2 * F, Kd, device="cuda", dtype=torch.bfloat16) * 0.02
    for _ in range(a.iters):
        K.gemm_swiglu_fwd(x, w)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
