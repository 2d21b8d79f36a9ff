#!/bin/bash
# A/B of the explicit PDL trigger: kernel timelines with both libraries.
out=gpurun_out/pdl_ab.jsonl; : > $out
for lib in "" notrig; do
  for c in "C1 1" "C1 8" "C2 1" "C3 1" "C4 1" "C5 1" "C5 4"; do
    if [ -n "$lib" ]; then export EB_LIB_PATH=paper_2206_08301_b200/lib/$lib/libeinplan_b200.so; else unset EB_LIB_PATH; fi
    python tools/kernel_timeline.py $c --out /tmp/tl.jsonl > /dev/null 2>gpurun_out/pdl_err.log || tail -3 gpurun_out/pdl_err.log
    python -c "import json,sys; l=json.loads(open('/tmp/tl.jsonl').read().splitlines()[-1]); print(json.dumps({'lib':'$lib' or 'trigger','cfg':'$c','span_us':round(l['span_us_per_run'],1),'gap_us':round(l['gap_us_per_run'],1)}))" >> $out
  done
done
cat $out
