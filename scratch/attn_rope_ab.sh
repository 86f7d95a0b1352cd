#!/bin/bash
out=gpurun_out/attn_rope; mkdir -p $out
export PYTHONPATH=$PWD
timeout 300 python scratch/attn_rope_ab.py > $out/ab.json 2> $out/ab.err; cat $out/ab.json; tail -3 $out/ab.err
