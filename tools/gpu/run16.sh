timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c5c.log 2>&1; echo rc=$?
tail -3 gpurun_out/c5c.log | cut -c1-300
