#!/bin/bash
out=gpurun_out/gemm_sweep4; rm -rf $out; mkdir -p $out
python -m pytest tests/test_kernels_gemm.py -q -x 2>&1 | tail -3 > $out/test.txt
run() {  # $1 tag, rest env
  tag=$1; shift
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 250 > $out/clk_$tag.csv &
  sp=$!
  env "$@" WARM=4 timeout 300 python scratch/gemm_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
  kill $sp
}
run cublas IMPL=cublas
run g8 GALV_GEMM_RASTER=8,0,0
run g16 GALV_GEMM_RASTER=16,0,0
run g8b GALV_GEMM_RASTER=8,0,0
cat $out/test.txt $out/sweep.jsonl
GALV_GEMM_RASTER=8,0,0 ONLY=gu_fwd WARM=0 REPS=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -c 1 -o $out/g8 python scratch/gemm_sweep.py > /dev/null 2>&1
