python -m pytest tests/test_gpu_parity.py -q -x -k "fused_redistribution or scatter or odd_extents or random_einsums or ttmc or c4" > gpurun_out/t7.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/t7.log
python -m pytest tests/test_multiprocess_gpu.py tests/test_full_size_all_p.py -q -x > gpurun_out/t7b.log 2>&1; echo "mp+full rc=$?"
tail -15 gpurun_out/t7b.log
timeout 900 python tools/push_ab.py gpurun_out/push_ab.jsonl > gpurun_out/push_ab.log 2>&1; echo "ab rc=$?"
tail -6 gpurun_out/push_ab.log
