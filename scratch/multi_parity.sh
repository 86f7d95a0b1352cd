#!/bin/bash
out=gpurun_out/multi2; mkdir -p $out
export PYTHONPATH=$PWD
timeout 1000 python -m pytest tests/test_multigpu.py -m gpu -x -q > $out/pytest_multigpu.log 2>&1; tail -1 $out/pytest_multigpu.log
