#!/bin/bash
# GEMM raster/hint sweep: sustained timing per variant + dram bytes of the gate|up fwd launch
out=gpurun_out/gemm_sweep; mkdir -p $out
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv > $out/smi_before.txt
for v in "16,0,0" "8,0,0" "32,0,0" "4,0,0" "16,0,1" "16,0,2" "16,0,4" "16,0,7" "32,0,7" "8,1,0" "16,0,0"; do
  GALV_GEMM_RASTER=$v timeout 300 python scratch/gemm_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
done
for v in "16,0,0" "32,0,0" "8,0,0" "16,0,1" "16,0,3" "32,0,3" "8,1,0"; do
  GALV_GEMM_RASTER=$v ONLY=gu_fwd,down_dgrad,gu_wgrad WARM=0 REPS=1 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_bf16 -c 6 --csv python scratch/gemm_sweep.py > $out/ncu_$v.csv 2>> $out/err.log
done
cat $out/sweep.jsonl
