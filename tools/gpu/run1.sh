set -x
free -g; nproc; nvidia-smi --query-gpu=name,memory.total --format=csv
python -m pytest tests/test_multiprocess_gpu.py -x -q > gpurun_out/mp.log 2>&1; echo "mp rc=$?"
tail -30 gpurun_out/mp.log
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu rc=$?"
tail -15 gpurun_out/gputests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench_c2.log
timeout 120 python bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_g2.log 2>&1; echo "g2 rc=$?"
tail -3 gpurun_out/bench_g2.log
