python -m pytest tests/test_gpu_parity.py -q -x -k "contract_ttm or c4 or fused_redistribution or odd_extents or random" > gpurun_out/t19.log 2>&1; echo "t rc=$?"; tail -3 gpurun_out/t19.log
python -m pytest tests/test_full_size_all_p.py -q -x -k "c4" > gpurun_out/t19b.log 2>&1; echo "full c4 rc=$?"; tail -2 gpurun_out/t19b.log
timeout 1500 python tools/scaling_proxy.py gpurun_out/scaling_proxy.jsonl > gpurun_out/sp.log 2>&1; echo "sp rc=$?"; grep '"C4"' gpurun_out/sp.log
