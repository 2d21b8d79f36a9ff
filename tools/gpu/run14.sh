mkdir -p gpurun_out/r14
timeout 300 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r14/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain -s 2 -c 1 -o gpurun_out/r14/chain python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r14/ncu.log 2>&1; echo "ncu rc=$?"
EB_CHAIN_TERMS=0 timeout 300 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r14/plain2.log 2>&1 && \
EB_CHAIN_TERMS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ttm2_ws -s 4 -c 1 -o gpurun_out/r14/ws python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r14/ncu2.log 2>&1; echo "ncu2 rc=$?"
for r in chain ws; do python tools/ncu_summary.py gpurun_out/r14/$r.ncu-rep gpurun_out/r14/$r.json > /dev/null 2>&1; ncu -i gpurun_out/r14/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/r14/${r}_sass.csv 2>/dev/null; gzip -f gpurun_out/r14/${r}_sass.csv; done
rm -f gpurun_out/r14/*.ncu-rep
ls -la gpurun_out/r14
