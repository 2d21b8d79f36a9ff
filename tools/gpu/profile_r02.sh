#!/bin/bash
# Round-2 ncu evidence with the final library: the launch list of the default
# bench command and one --set full capture per configuration's dominant
# kernel.  Every capture runs only after the same command exited 0 without
# ncu.  Reports are condensed on the box (tools/ncu_summary.py + SASS source
# page) and the large .ncu-rep files dropped.
set -u
O=gpurun_out/prof2
mkdir -p $O
NCU="ncu --clock-control none"
run() {  # name, kernel regex, count, command...
  local name=$1 rx=$2 c=$3; shift 3
  if timeout 600 "$@" > $O/${name}_plain.log 2>&1; then
    timeout 900 $NCU --set full --import-source on -k regex:$rx -c $c -o $O/ncu_${name}_r02 "$@" \
      > $O/ncu_${name}.log 2>&1
    echo "$name ncu rc=$?"
  else
    echo "$name plain run failed"; tail -5 $O/${name}_plain.log
  fi
}
# 1) launch list of the bench command (cold, serialised per-launch durations)
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs"
if timeout 600 $B > $O/launches_plain.log 2>&1; then
  timeout 900 $NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/launches_c2_bench_r02.csv \
    $B > $O/launches.log 2>&1; echo "launch list rc=$?"
fi
# 2) dominant kernels
run c2m0 contract_kernel 1 python tools/prof_contract.py c2m0 2
run c2m2 contract_kernel 1 python tools/prof_contract.py c2m2 2
run c1 contract_kernel 1 python tools/prof_contract.py c1 2
run c3 mttkrp_rf 1 python tools/prof_contract.py c3 2
run c5 ttm2_ws 2 python tools/ttm2_bench.py 1
for r in $O/*.ncu-rep; do
  python tools/ncu_summary.py $r ${r%.ncu-rep}.json > /dev/null 2>&1
  ncu -i $r --page source --csv --print-source sass > ${r%.ncu-rep}_sass.csv 2>/dev/null
  gzip -f ${r%.ncu-rep}_sass.csv
  rm -f $r
done
ls -la $O
