#!/bin/bash
# Bench lines of every BASELINE config with the final library, plus the
# reference arm of the default config.
: > gpurun_out/bench_configs.jsonl
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log >> gpurun_out/bench_configs.jsonl
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_reference.jsonl
cut -c1-300 gpurun_out/bench_configs.jsonl gpurun_out/bench_reference.jsonl
