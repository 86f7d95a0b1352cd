#!/bin/bash
out=gpurun_out/gemm_sweep2; mkdir -p $out
run() {  # $1 tag, rest env
  tag=$1; shift
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 250 > $out/clk_$tag.csv &
  sp=$!
  env "$@" WARM=4 timeout 300 python scratch/gemm_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
  kill $sp
}
run cublas IMPL=cublas
run g16 GALV_GEMM_RASTER=16,0,0
run g8 GALV_GEMM_RASTER=8,0,0
run g16n GALV_GEMM_RASTER=16,1,0
run g16n1 GALV_GEMM_RASTER=16,1,1
run cublas2 IMPL=cublas
run g8b GALV_GEMM_RASTER=8,0,0
cat $out/sweep.jsonl
for f in $out/clk_*.csv; do echo $f; awk -F', ' '{print $1}' $f | sort -n | awk '{a[NR]=$1} END{print "median", a[int(NR/2)]}'; done
