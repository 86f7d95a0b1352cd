#!/bin/bash
python bench.py --model gpt2-medium --seqs-per-gpu 16 --no-cpu-baseline --cluster-profile profiles/b200_cluster_gpt2m.json > gpurun_out/c2d.jsonl 2>gpurun_out/c2d.err
python -c "
import json; d=json.loads(open('gpurun_out/c2d.jsonl').read().strip().splitlines()[-1]); r=d['roofline']; print('c2', round(d['value']), d['ms_per_step'], d['mfu'], d['prediction_error'], d['clocks']['sm_mhz'], round(r['achieved']), d['gpu_launches'])"
python -m pytest tests/test_runtime_parity.py -q -x 2>&1 | tail -1
