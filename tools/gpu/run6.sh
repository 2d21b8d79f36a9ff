# round-2 evidence: bench lines for every config, the headline line, GEMM ncu capture
mkdir -p gpurun_out/r02
for c in C1 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02/bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/r02/bench_$c.log | cut -c1-400
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_C2.log 2>&1; echo "bench C2 rc=$?"
tail -1 gpurun_out/r02/bench_C2.log | cut -c1-600
timeout 600 python tools/gemm_chain_check.py --only 1MM --reps 1 > gpurun_out/r02/gemm_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_kernel -s 2 -c 1 -o gpurun_out/r02/ncu_gemm python tools/gemm_chain_check.py --only 1MM --reps 1 > gpurun_out/r02/ncu_gemm.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/r02/ncu_gemm.ncu-rep gpurun_out/r02/ncu_gemm.json > /dev/null 2>&1
ncu -i gpurun_out/r02/ncu_gemm.ncu-rep --page source --csv --print-source sass > gpurun_out/r02/ncu_gemm_sass.csv 2>/dev/null; gzip -f gpurun_out/r02/ncu_gemm_sass.csv
ls -la gpurun_out/r02
