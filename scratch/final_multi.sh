#!/bin/bash
# 4-GPU box: multi-GPU parity suite, then N=2 / N=4 headline and C5 / C4 with the current kernels
out=gpurun_out/fmulti; mkdir -p $out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -x -q > $out/pytest_mgpu.log 2>&1; tail -1 $out/pytest_mgpu.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$TR --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 --no-cpu-baseline > $out/n2.jsonl 2> $out/n2.err
$TR --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 --no-cpu-baseline > $out/n4.jsonl 2> $out/n4.err
$TR --nproc-per-node 4 --master-port 29603 bench.py --gpus 4 --model llama2-13b --seqs-per-gpu 2 --steps 2 --warmup 3 --cluster-profile profiles/b200_cluster_llama13b.json --no-cpu-baseline > $out/c5.jsonl 2> $out/c5.err
for f in n2 n4 c5; do echo $f; grep -o "\"value\": [0-9.]*\|prediction_error\": [-0-9.e]*\|sm_mhz\": [0-9.]*\|\"mfu\": [0-9.]*" $out/$f.jsonl | tr "\n" " "; echo; done
