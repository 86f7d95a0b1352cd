#!/bin/bash
python -m pytest tests/test_kernels_gemm.py -q -x 2>&1 | tail -1
for v in 8,0,0 8,0,32 8,0,0 8,0,32; do
  GALV_GEMM_RASTER=$v WARM=4 python scratch/gemm_sweep.py
done
