timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or ttmc_o5" > gpurun_out/t10.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/t10.log
timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"
tail -1 gpurun_out/c5.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); r=l['roofline']; print(l['value'], l['ms_per_step'], r['frac'], r['kernel_ms_per_launch'], r['kernel_launches_timed'], l['clocks'])"
