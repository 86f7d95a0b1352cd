#!/bin/bash
# Re-entry check after the container rebuild: GPU suite, smoke, default bench x2, launch list
out=gpurun_out/final_check; mkdir -p $out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; tail -1 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
for i in 1 2; do timeout 600 python bench.py > $out/bench_n1_$i.jsonl 2> $out/bench_n1_$i.err; tail -1 $out/bench_n1_$i.jsonl | cut -c1-400; done
timeout 600 python bench.py --impl reference > $out/bench_ref.jsonl 2> $out/bench_ref.err; tail -1 $out/bench_ref.jsonl | cut -c1-300
