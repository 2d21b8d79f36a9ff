#!/bin/bash
# ncu evidence for one round (run on the GPU box through gpurun; each capture
# only after the same command ran clean without ncu).  Reports land in
# gpurun_out/; tools/ncu_summary.py condenses them into profiles/.
set -u
O=gpurun_out/prof
mkdir -p $O
NCU="ncu --clock-control none"
# 1) launch list of the bench command itself (per-launch durations, cold, serialised)
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches_bench.log 2>&1
# 2) full captures of the dominant kernel per configuration
for c in c2m0 c2m1 c2m2 c2pair c1; do
  timeout 600 $NCU --set full --import-source on -k regex:contract_kernel -c 1 -o $O/ncu_$c \
    python tools/prof_contract.py $c 2 > $O/ncu_$c.log 2>&1
done
timeout 600 $NCU --set full --import-source on -k regex:mttkrp_rf -c 1 -o $O/ncu_c3 \
  python tools/prof_contract.py c3 2 > $O/ncu_c3.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ttm2 -c 2 -o $O/ncu_c5_ttm2 \
  python tools/ttm2_bench.py 1 > $O/ncu_c5.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:contract_kernel -c 2 -o $O/ncu_c4 \
  python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c4.log 2>&1

# condense on the box (the reports are too large to bring back whole)
for r in $O/*.ncu-rep; do
  python tools/ncu_summary.py $r ${r%.ncu-rep}.json > /dev/null 2>&1
  ncu -i $r --page source --csv --print-source sass > ${r%.ncu-rep}_sass.csv 2>/dev/null
  gzip -f ${r%.ncu-rep}_sass.csv
done
ls -la $O
du -sh $O
# keep only the small reports
for r in $O/*.ncu-rep; do [ $(stat -c %s $r) -gt 6000000 ] && rm -f $r; done
du -sh gpurun_out
