mkdir -p gpurun_out/r22
timeout 600 python tools/c5p4_prof.py > gpurun_out/r22/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ttm2_ws -c 8 -o gpurun_out/r22/c5p4 python tools/c5p4_prof.py > gpurun_out/r22/ncu.log 2>&1; echo "ncu1 rc=$?"
timeout 600 python tools/c4p8_launches.py 8 > gpurun_out/r22/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:contract_kernel -s 16 -c 2 -o gpurun_out/r22/c4p8 python tools/c4p8_launches.py 8 > gpurun_out/r22/ncu2.log 2>&1; echo "ncu2 rc=$?"
for r in c5p4 c4p8; do python tools/ncu_summary.py gpurun_out/r22/$r.ncu-rep gpurun_out/r22/$r.json > /dev/null 2>&1; ncu -i gpurun_out/r22/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/r22/${r}_sass.csv 2>/dev/null; gzip -f gpurun_out/r22/${r}_sass.csv; done
rm -f gpurun_out/r22/*.ncu-rep; ls gpurun_out/r22
