#!/bin/bash
# inverse RoPE fused into the attention backward epilogues: GPU tests, then N=1 bench A/B
out=gpurun_out/rope_bwd; mkdir -p $out
export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_kernels_attn.py -m gpu -x -q > $out/pytest_attn.log 2>&1; tail -1 $out/pytest_attn.log
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; tail -1 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $out/fused_$i.jsonl 2>&1
  GALV_ROPE_UNFUSED=1 timeout 600 python bench.py --no-cpu-baseline > $out/unfused_$i.jsonl 2>&1
done
for f in $out/*.jsonl; do echo $f; grep -o "\"value\": [0-9.]*\|sm_mhz\": [0-9.]*\|gpu_launches\": [0-9]*" $f | tr "\n" " "; echo; done
