#!/bin/bash
# RoPE-in-QKV-epilogue: GPU tests, then N=1 bench A/B (GALV_ROPE_UNFUSED=1 = GEMM + RoPE kernel)
out=gpurun_out/rope; mkdir -p $out
export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_kernels_gemm.py -m gpu -x -q -k rope > $out/pytest_rope.log 2>&1; tail -1 $out/pytest_rope.log
timeout 600 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; tail -1 $out/pytest_gpu.log
for i in 1 2; do
  python bench.py --no-cpu-baseline > $out/fused_$i.jsonl 2>&1
  GALV_ROPE_UNFUSED=1 python bench.py --no-cpu-baseline > $out/unfused_$i.jsonl 2>&1
done
for f in $out/*.jsonl; do echo $f; grep -o "\"value\": [0-9.]*\|sm_mhz\": [0-9.]*\|gemm_launches\": [0-9]*" $f | tr "\n" " "; echo; done
