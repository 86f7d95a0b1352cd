#!/usr/bin/env python
"""Same-box attention A/B: galv tcgen05 kernels vs the library paths on this B200.

    python tools/attn_ab.py [--out profiles/r02/attn_ab.jsonl]

Causal bf16 attention, head_dim 128, inputs as the runtime lays them out (strided q/k/v
views of one [B, S, 3, H, D] qkv buffer).  Each arm is timed with CUDA events on the
launching stream (warm-up, then the median of `--iters` launches).  FLOPs counted causal:
fwd 2*B*H*S^2*D (QK^T + PV over the lower triangle), bwd 2.5x fwd (5 GEMM-equivalents);
the term the kernels realize is the cost model's flops_per_token_sq (ref costmodel.py:104).

Arms: galv fwd / bwd / bwd+inverse-RoPE; torch SDPA with the cuDNN backend (fwd, and
fwd+bwd through autograd -> bwd = difference); torch SDPA flash backend; flash_attn 2.x;
flashinfer single_prefill (fwd only).  An arm that cannot run here records its error.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, iters=20, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    return statistics.median(out)


def run_shape(B, S, H, D, iters, libs=True):
    from paper_2504_21411_b200 import kernels as K
    dev = "cuda"
    torch.manual_seed(0)
    qkv = torch.randn(B, S, 3, H, D, device=dev).bfloat16()
    q, k, v = qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]
    o = torch.empty(B, S, H, D, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(B, H, S, device=dev)
    do = torch.randn(B, S, H, D, device=dev).bfloat16()
    dqkv = torch.empty_like(qkv)
    scale = 1 / math.sqrt(D)
    ws = torch.empty(K.attn_bwd_workspace_bytes(B, S, H, D, torch.bfloat16), dtype=torch.uint8,
                     device=dev)
    f_fwd = 2.0 * B * H * S * S * D  # causal: half of 4*B*H*S^2*D
    f_bwd = 2.5 * f_fwd
    rows = []

    def rec(arm, phase, us, flops, note=""):
        rows.append({"shape": f"B{B} S{S} H{H} D{D} causal", "arm": arm, "phase": phase,
                     "us": us, "tflops": flops / (us * 1e-6) / 1e12 if us else None,
                     "note": note})

    us = timed(lambda: K.attn_fwd(q, k, v, o, lse, scale=scale, causal=True), iters)
    rec("galv", "fwd", us, f_fwd)
    us = timed(lambda: K.attn_bwd(q, k, v, o, do, lse, dqkv[:, :, 0], dqkv[:, :, 1],
                                  dqkv[:, :, 2], scale=scale, causal=True, workspace=ws), iters)
    rec("galv", "bwd", us, f_bwd)
    if D == 128:
        us = timed(lambda: K.attn_bwd(q, k, v, o, do, lse, dqkv[:, :, 0], dqkv[:, :, 1],
                                      dqkv[:, :, 2], scale=scale, causal=True, workspace=ws,
                                      rope_theta=10000.0), iters)
        rec("galv", "bwd+inverse_rope", us, f_bwd)

    if not libs:
        return rows
    from torch.nn.attention import SDPBackend, sdpa_kernel
    import torch.nn.functional as F
    qt, kt, vt = (t.transpose(1, 2) for t in (q, k, v))  # [B, H, S, D] strided views
    for name, be in (("torch_sdpa_cudnn", SDPBackend.CUDNN_ATTENTION),
                     ("torch_sdpa_flash", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                us_f = timed(lambda: F.scaled_dot_product_attention(qt, kt, vt, is_causal=True),
                             iters)
                qg, kg, vg = (t.detach().clone().requires_grad_(True) for t in (qt, kt, vt))
                dot = do.transpose(1, 2)

                def fb():
                    out = F.scaled_dot_product_attention(qg, kg, vg, is_causal=True)
                    out.backward(dot)
                us_fb = timed(fb, iters)
            rec(name, "fwd", us_f, f_fwd)
            rec(name, "bwd", us_fb - us_f, f_bwd, "fwd+bwd through autograd minus fwd")
        except Exception as exc:  # noqa: BLE001
            rec(name, "fwd", None, f_fwd, f"unavailable: {type(exc).__name__}: {exc}"[:300])
    try:
        from flash_attn import flash_attn_func
        us_f = timed(lambda: flash_attn_func(q, k, v, causal=True), iters)
        qg, kg, vg = (t.detach().clone().requires_grad_(True) for t in (q, k, v))

        def fb2():
            flash_attn_func(qg, kg, vg, causal=True).backward(do)
        us_fb = timed(fb2, iters)
        rec("flash_attn2", "fwd", us_f, f_fwd)
        rec("flash_attn2", "bwd", us_fb - us_f, f_bwd, "fwd+bwd through autograd minus fwd")
    except Exception as exc:  # noqa: BLE001
        rec("flash_attn2", "fwd", None, f_fwd, f"unavailable: {type(exc).__name__}: {exc}"[:300])
    try:
        import flashinfer
        if B == 1:
            qs, ks, vs = q[0], k[0], v[0]  # [S, H, D] (NHD)
            us_f = timed(lambda: flashinfer.single_prefill_with_kv_cache(
                qs, ks, vs, causal=True), iters)
            rec("flashinfer_single_prefill", "fwd", us_f, f_fwd)
        else:
            qs = q.reshape(B * S, H, D)
            ks, vs = k.reshape(B * S, H, D), v.reshape(B * S, H, D)
            indptr = torch.arange(0, (B + 1) * S, S, device=dev, dtype=torch.int32)
            w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(
                torch.empty(256 << 20, dtype=torch.uint8, device=dev), "NHD")
            w.plan(indptr, indptr, H, H, D, causal=True, q_data_type=torch.bfloat16)
            us_f = timed(lambda: w.run(qs, ks, vs), iters)
            rec("flashinfer_batch_prefill_ragged", "fwd", us_f, f_fwd)
    except Exception as exc:  # noqa: BLE001
        rec("flashinfer", "fwd", None, f_fwd, f"unavailable: {type(exc).__name__}: {exc}"[:300])
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--shapes", default="2x4096x32,1x32768x8,4x1024x16x64")
    ap.add_argument("--galv-only", action="store_true", help="skip the library arms")
    ap.add_argument("--lib", default=None, help="load this libgalv build instead (A/B)")
    args = ap.parse_args()
    if args.lib:
        from paper_2504_21411_b200 import kernels as K
        K._lib = K.load_library(args.lib)
    rows = []
    for spec in args.shapes.split(","):
        parts = [int(x) for x in spec.split("x")]
        B, S, H = parts[:3]
        D = parts[3] if len(parts) > 3 else 128
        rows += run_shape(B, S, H, D, args.iters, libs=not args.galv_only)
    for r in rows:
        print(json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
