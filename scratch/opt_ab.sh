#!/bin/bash
for v in 1 0 1 0; do
  GALV_OPT_SIDE_STREAM=$v python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/opt_$v.jsonl 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/opt_$v.jsonl').read().strip().splitlines()[-1]); print('side=$v', round(d['value']), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],2), round(d['roofline']['achieved']))"
done
