b() { timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/c5x.log 2>&1; tail -1 gpurun_out/c5x.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); r=l['roofline']; print(round(l['ms_per_step'],4), round(r['frac'],3), l['clocks']['sm_mhz'])"; }
echo -n "chain: "; EB_CHAIN_TERMS=1 b
echo -n "chain A-only probe: "; EB_CHAIN_TERMS=1 EB_CHAIN_FLAGS=15 b
echo -n "two launches: "; b
