#!/usr/bin/env python
"""HBM-bound kernels of the GPT-2-medium step at its shapes (16 x 1024 tokens): CUDA events
over 50 calls each, achieved GB/s on the algorithmic bytes.  Env switches the library reads
once per process (GALV_NORM_WARP=0, GALV_NORM_UNFUSED=1) select the A/B variants.

    python tools/pointwise_bench.py [--out FILE]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    from paper_2504_21411_b200 import kernels as K
    bf = torch.bfloat16
    res = {"env": {k: os.environ.get(k) for k in ("GALV_NORM_WARP", "GALV_NORM_UNFUSED",
                                                  "GALV_NORM_NARROW")}}
    for rows, cols, layer in [(16384, 1024, True), (16384, 1024, False), (8192, 4096, False),
                              (16384, 2048, True), (16384, 768, True), (16384, 512, True)]:
        x = torch.randn(rows, cols, device="cuda", dtype=bf)
        g = torch.randn(cols, device="cuda", dtype=bf)
        b = torch.randn(cols, device="cuda", dtype=bf)
        dy, dres, dx = torch.randn_like(x), torch.randn_like(x), torch.empty_like(x)
        dg, db = torch.zeros(cols, device="cuda"), torch.zeros(cols, device="cuda")
        if layer:
            _, mean, rstd = K.layernorm_fwd(x, g, b, 1e-5)
            fn = lambda: K.layernorm_bwd(x, g, mean, rstd, dy, dg, db, dres=dres, dx=dx)
        else:
            _, rstd = K.rmsnorm_fwd(x, g, 1e-5)
            fn = lambda: K.rmsnorm_bwd(x, g, rstd, dy, dg, dres=dres, dx=dx)
        us = timed(fn)
        res[f"{'ln' if layer else 'rms'}_bwd_{rows}x{cols}"] = {
            "us": round(us, 1), "GBps": round(4 * rows * cols * 2 / us / 1e3)}
    T, F = 16384, 4096
    pre = torch.randn(T, F, device="cuda", dtype=bf)
    bias = torch.randn(F, device="cuda", dtype=bf)
    us = timed(lambda: K.bias_gelu_fwd(pre, bias))
    res["bias_gelu_fwd_16384x4096"] = {"us": round(us, 1), "GBps": round(2 * T * F * 2 / us / 1e3)}
    dact = torch.randn_like(pre)
    acc = torch.zeros(F, device="cuda")
    us = timed(lambda: K.bias_gelu_bwd_colsum(pre, bias, dact, acc))
    res["bias_gelu_bwd_colsum_16384x4096"] = {"us": round(us, 1),
                                              "GBps": round(3 * T * F * 2 / us / 1e3)}
    for n in (1024, 3072):
        m = torch.randn(T, n, device="cuda", dtype=bf)
        o = torch.zeros(n, device="cuda")
        us = timed(lambda: K.colsum(m, o))
        res[f"colsum_16384x{n}"] = {"us": round(us, 1), "GBps": round(T * n * 2 / us / 1e3)}
    V = 50304
    logits = torch.randn(T, V, device="cuda", dtype=bf)
    labels = torch.randint(0, V, (T,), device="cuda")
    st, loss = torch.empty(T, 3, device="cuda"), torch.empty(T, device="cuda")
    us = timed(lambda: K.xent(logits, labels, st, 3, loss=loss, dlogits=logits,
                              grad_scale=1.0 / T), n=10)
    res[f"xent_16384x{V}"] = {"us": round(us, 1), "GBps": round(2 * T * V * 2 / us / 1e3)}
    print(json.dumps(res))
    if args.out:
        with open(args.out, "a") as fh:
            fh.write(json.dumps(res) + "\n")


if __name__ == "__main__":
    main()
