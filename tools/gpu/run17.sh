for c in "C2 2" "C4 4" "C5 4"; do set -- $c
  timeout 900 python bench.py --config $1 --gpus $2 --share-gpu --steps 3 --warmup 3 --no-e2e > gpurun_out/share_$1.log 2>&1; echo "$1 x$2 rc=$?"
  grep '"metric"' gpurun_out/share_$1.log | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['n_gpus'], l['config']['transport'], l['config'].get('grids'), l['ms_per_step'], l['config'].get('shared_gpu','')[:30])"
  grep -i "error\|Traceback" gpurun_out/share_$1.log | head -5
done
