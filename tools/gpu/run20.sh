mkdir -p gpurun_out/r20
timeout 600 python tools/c5p4_prof.py > gpurun_out/r20/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:ttm2_ws -c 10 -o gpurun_out/r20/c5p4 python tools/c5p4_prof.py > gpurun_out/r20/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/r20/c5p4.ncu-rep gpurun_out/r20/c5p4.json > /dev/null 2>&1
rm -f gpurun_out/r20/*.ncu-rep
