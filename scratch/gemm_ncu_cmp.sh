#!/bin/bash
out=gpurun_out/gemm_cmp; mkdir -p $out
for s in gu_fwd o_wgrad; do
IMPL=cublas ONLY=$s WARM=0 REPS=1 timeout 300 ncu --set full --clock-control none -k regex:'nvjet|gemm|sm100|cutlass|Kernel' -c 1 -o $out/cublas_$s python scratch/gemm_sweep.py > $out/cublas_$s.log 2>&1
ONLY=$s WARM=0 REPS=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -c 1 -o $out/galv_$s python scratch/gemm_sweep.py > $out/galv_$s.log 2>&1
done
ls -la $out
