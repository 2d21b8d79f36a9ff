b() { timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c5x.log 2>&1; tail -1 gpurun_out/c5x.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); r=l['roofline']; print(round(l['ms_per_step'],4), round(r['frac'],3), l['clocks']['sm_mhz'])"; }
echo -n "chain off: "; EB_CHAIN_TERMS=0 b
for lag in 1 2 4 8; do echo -n "lag=$lag: "; EB_CHAIN_LAG=$lag b; done
echo -n "chain off: "; EB_CHAIN_TERMS=0 b
