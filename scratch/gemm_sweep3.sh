#!/bin/bash
out=gpurun_out/gemm_sweep3; mkdir -p $out
run() {  # $1 tag, rest env
  tag=$1; shift
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 250 > $out/clk_$tag.csv &
  sp=$!
  env "$@" WARM=4 timeout 300 python scratch/gemm_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
  kill $sp
}
run cublas IMPL=cublas
run old GALV_GEMM_RASTER=8,0,8
run new GALV_GEMM_RASTER=8,0,0
run new16 GALV_GEMM_RASTER=8,0,16
run new16g GALV_GEMM_RASTER=16,0,16
run old2 GALV_GEMM_RASTER=8,0,8
run new2 GALV_GEMM_RASTER=8,0,0
cat $out/sweep.jsonl
for f in $out/clk_*.csv; do echo $f; awk -F', ' '{print $1}' $f | sort -n | awk '{a[NR]=$1} END{print "median", a[int(NR/2)]}'; done
for v in 8,0,0 8,0,16; do
GALV_GEMM_RASTER=$v ONLY=gu_fwd WARM=0 REPS=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -c 1 -o $out/galv_gu_fwd_$v python scratch/gemm_sweep.py > /dev/null 2>&1
done
