#!/bin/bash
# multi-GPU parity suite + N=2/N=4/C5/C4 benches with the fused RoPE backward
out=gpurun_out/multi; mkdir -p $out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -x -q > $out/pytest_multigpu.log 2>&1; tail -1 $out/pytest_multigpu.log
timeout 1500 bash scratch/multi_bench.sh
