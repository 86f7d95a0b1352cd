#!/bin/bash
out=gpurun_out/attnvar; mkdir -p $out
for i in 1 2; do
python scratch/attn_sustained.py
GALV_LIB=$PWD/scratch/libgalv_attn_suspend.so python scratch/attn_sustained.py
done
for v in default suspend default suspend; do
  if [ $v = suspend ]; then export GALV_LIB=$PWD/scratch/libgalv_attn_suspend.so; else unset GALV_LIB; fi
  python bench.py --no-cpu-baseline --steps 4 --warmup 3 > $out/b_$v.jsonl 2>/dev/null
  python -c "
import json; d=json.loads(open('$out/b_$v.jsonl').read().strip().splitlines()[-1]); print('$v', round(d['value']), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],2))"
done
