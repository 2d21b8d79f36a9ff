for f in 7 6 4 2 0; do
  EB_CHAIN_FLAGS=$f timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c5_$f.log 2>&1
  echo -n "flags=$f "; tail -1 gpurun_out/c5_$f.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); r=l['roofline']; print(round(l['ms_per_step'],4), round(r['frac'],3), l['clocks']['sm_mhz'])"
done
EB_CHAIN_TERMS=0 timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c5_off.log 2>&1
echo -n "chain off "; tail -1 gpurun_out/c5_off.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); r=l['roofline']; print(round(l['ms_per_step'],4), round(r['frac'],3), l['clocks']['sm_mhz'])"
