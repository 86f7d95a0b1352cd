#!/bin/bash
out=gpurun_out/launches; mkdir -p $out
export PYTHONPATH=$PWD
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 10000 --csv --log-file $out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu.log 2>&1; echo rc $?
gzip -f $out/launches.csv
python scratch/launch_share.py $out/launches.csv.gz | head -30
