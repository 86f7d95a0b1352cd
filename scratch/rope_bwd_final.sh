#!/bin/bash
out=gpurun_out/rope_bwd2; mkdir -p $out
export PYTHONPATH=$PWD
timeout 300 python scratch/attn_rope_ab.py > $out/ab.json 2> $out/ab.err; cat $out/ab.json
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; tail -1 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 600 python bench.py > $out/bench_n1.jsonl 2> $out/bench_n1.err
grep -o "\"value\": [0-9.]*\|sm_mhz\": [0-9.]*\|gpu_launches\": [0-9]*\|prediction_error\": [-0-9.]*" $out/bench_n1.jsonl | tr "\n" " "; echo
