#!/bin/bash
out=gpurun_out/c4mg; mkdir -p $out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$TR --nproc-per-node 4 --master-port 29631 bench.py --gpus 4 --model gpt-1.3b --seqs-per-gpu 16 --layer-pattern tp4,dp4z3,tp2dp2 --microbatch 8 --steps 3 --warmup 3 --no-cpu-baseline > $out/c4.jsonl 2> $out/c4.err
python -c "
import json; d=json.loads([l for l in open('$out/c4.jsonl') if l.startswith('{')][-1]); print('c4', round(d['value']), d['mfu'], d['prediction_error'], d['clocks']['sm_mhz'], d['config']['parallelism'])"
python -m pytest tests/test_multigpu.py -x -q > $out/mgpu.log 2>&1; echo "mgpu rc=$?"; tail -2 $out/mgpu.log
