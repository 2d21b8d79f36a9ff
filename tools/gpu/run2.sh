python -m pytest tests/test_multiprocess_gpu.py -x -q > gpurun_out/mp.log 2>&1; echo "mp rc=$?"
tail -5 gpurun_out/mp.log
python -m pytest tests/test_full_size_all_p.py -q --durations=30 > gpurun_out/full.log 2>&1; echo "full rc=$?"
tail -45 gpurun_out/full.log
timeout 900 python tools/gemm_chain_check.py --out gpurun_out/gemm_chain.jsonl > gpurun_out/gemm.log 2>&1; echo "gemm rc=$?"
tail -5 gpurun_out/gemm.log
timeout 600 python bench.py --impl reference --steps 8 --warmup 0 > gpurun_out/ref_c2.log 2>&1; echo "ref rc=$?"
tail -2 gpurun_out/ref_c2.log | cut -c1-3000
