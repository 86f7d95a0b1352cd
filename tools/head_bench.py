#!/usr/bin/env python
"""LM head (final norm + vocab GEMM + cross-entropy + dgrad + wgrad) timing by chunk count.

    python tools/head_bench.py [--tokens 8192] [--chunks 1,2,4]

Times Head.forward_backward (runtime/layers.py) at Llama-2-7B width (h 4096, V 32000) on
one GPU with CUDA events, and every GEMM of one call (kernels.KernelStats(time_gemm))."""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--chunk-bytes", default="1073741824,268435456")
    ap.add_argument("--model", default="llama2-7b")
    args = ap.parse_args()
    from paper_2504_21411_b200 import kernels as K
    from paper_2504_21411_b200.planner.strategy import ParallelStrategy
    from paper_2504_21411_b200.runtime import layers
    from paper_2504_21411_b200.runtime.config import MODEL_PRESETS, HybridConfig
    from paper_2504_21411_b200.runtime.topology import Topology
    cfg = MODEL_PRESETS[args.model]
    s = ParallelStrategy(1, 1, 0, False, False)
    hc = HybridConfig(pp=1, microbatch=1, n_microbatches=1, stage_ranges=((0, 1),),
                      layer_strategies=(s,))
    dev = torch.device("cuda", 0)
    head = layers.Head(cfg, s, Topology(hc, rank=0, world=1), dtype=torch.bfloat16,
                       grad_dtype=torch.bfloat16, device=dev)
    head.store.load({n: 0.02 * torch.randn(shp) for n, (_, shp) in head.store.layout.items()})
    T = args.tokens
    x = torch.randn(T, cfg.hidden, device=dev, dtype=torch.bfloat16)
    labels = torch.randint(0, cfg.vocab, (T,), device=dev)
    flops = 3 * 2.0 * T * cfg.hidden * cfg.vocab
    layers.HEAD_CHUNK_MIN_ROWS = 128
    for c in [int(v) for v in args.chunk_bytes.split(",")]:
        layers.HEAD_CHUNK_BYTES = c
        for _ in range(3):
            head.forward_backward(x, labels, 1.0 / T)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            head.forward_backward(x, labels, 1.0 / T)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        st = K.start_stats(time_gemm=True)
        head.forward_backward(x, labels, 1.0 / T)
        K.stop_stats()
        g = st.gemm_summary()
        shapes = [(shp, round(s0.elapsed_time(s1) * 1e3, 1)) for _, s0, s1, shp in st.gemm_events]
        print(json.dumps({"chunk_bytes": c, "tokens": T, "ms": ms, "tflops_gemm_flops": flops / ms / 1e9,
                          "gemm_ms": g["ms"], "gemm_tflops": g["tflops"],
                          "gemms_us": shapes[:6]}), flush=True)


if __name__ == "__main__":
    main()
