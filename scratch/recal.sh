#!/bin/bash
# recalibrate the cluster profiles with the current kernels, then re-run the benches on them
out=gpurun_out/recal; mkdir -p $out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$TR --nproc-per-node 4 --master-port 29611 -m paper_2504_21411_b200.profiler -o $out/b200_cluster.json --model llama2-7b --microbatch 2 > $out/prof7b.log 2>&1
python -m paper_2504_21411_b200.profiler -o $out/b200_cluster_llama13b.json --model llama2-13b --microbatch 1 --table-from $out/b200_cluster.json > $out/prof13b.log 2>&1
python -m paper_2504_21411_b200.profiler -o $out/b200_cluster_gpt2m.json --model gpt2-medium --microbatch 16 --table-from $out/b200_cluster.json > $out/profg.log 2>&1
$TR --nproc-per-node 2 --master-port 29612 bench.py --gpus 2 --no-cpu-baseline --cluster-profile $out/b200_cluster.json > $out/n2.jsonl 2> $out/n2.err
$TR --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --no-cpu-baseline --cluster-profile $out/b200_cluster.json > $out/n4.jsonl 2> $out/n4.err
$TR --nproc-per-node 4 --master-port 29614 bench.py --gpus 4 --model llama2-13b --seqs-per-gpu 2 --steps 2 --warmup 2 --no-cpu-baseline --cluster-profile $out/b200_cluster_llama13b.json > $out/c5.jsonl 2> $out/c5.err
python bench.py --no-cpu-baseline --cluster-profile $out/b200_cluster.json > $out/n1.jsonl 2> $out/n1.err
python bench.py --model gpt2-medium --seqs-per-gpu 16 --no-cpu-baseline --cluster-profile $out/b200_cluster_gpt2m.json > $out/c2.jsonl 2> $out/c2.err
for f in n1 n2 n4 c5 c2; do python -c "
import json; d=json.loads([l for l in open('$out/$f.jsonl') if l.startswith('{')][-1]); print('$f', round(d['value']), round(d['mfu'],4), round(d['prediction_error'],4), d['clocks']['sm_mhz'], d['config']['parallelism'], d.get('peak_mem_gb'))" 2>&1 | tail -1; done
grep -h device_flops $out/*.meta.json
