#!/bin/bash
# C5 (4 GPUs) and C2 (1 GPU) with bench.py's per-model default cluster profiles
out=gpurun_out/c5c2; mkdir -p $out
export PYTHONPATH=$PWD
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29603 bench.py --gpus 4 --model llama2-13b --seqs-per-gpu 2 --steps 2 --warmup 3 --no-cpu-baseline > $out/c5.jsonl 2> $out/c5.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --model gpt2-medium --seqs-per-gpu 16 --no-cpu-baseline > $out/c2.jsonl 2> $out/c2.err
for f in c5 c2; do python -c "
import json; d=json.loads([l for l in open('$out/$f.jsonl') if l.startswith('{')][-1]); print('$f', round(d['value']), d['mfu'], d['prediction_error'], d['clocks']['sm_mhz'], d['config']['parallelism'], d['cluster_profile'])" 2>&1 | tail -1; done
