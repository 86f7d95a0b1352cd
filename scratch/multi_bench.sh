#!/bin/bash
# N=2 / N=4 headline + C5 / C4 on one 4-GPU box
out=gpurun_out/multi; mkdir -p $out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$TR --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 --no-cpu-baseline > $out/n2.jsonl 2> $out/n2.err
$TR --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 --no-cpu-baseline > $out/n4.jsonl 2> $out/n4.err
$TR --nproc-per-node 4 --master-port 29603 bench.py --gpus 4 --model llama2-13b --seqs-per-gpu 2 --steps 2 --warmup 2 --no-cpu-baseline > $out/c5.jsonl 2> $out/c5.err
$TR --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 --model gpt-1.3b --seqs-per-gpu 16 --layer-pattern tp4,dp4z3,tp2dp2 --microbatch 8 --steps 3 --warmup 3 --no-cpu-baseline > $out/c4.jsonl 2> $out/c4.err
for f in n2 n4 c5 c4; do python -c "
import json; d=json.loads([l for l in open('$out/$f.jsonl') if l.startswith('{')][-1]); print('$f', round(d['value']), d['mfu'], d['prediction_error'], d['clocks']['sm_mhz'], d['config']['parallelism'], d.get('peak_mem_gb'))" 2>&1 | tail -1; done
