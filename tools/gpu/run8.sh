python -m pytest tests/test_gpu_parity.py -q -x -k "fused_redistribution or scatter or ttmc or c4 or c5" > gpurun_out/t8.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/t8.log
timeout 900 python tools/push_ab.py gpurun_out/push_ab.jsonl > gpurun_out/push_ab.log 2>&1; echo "ab rc=$?"
tail -6 gpurun_out/push_ab.log
