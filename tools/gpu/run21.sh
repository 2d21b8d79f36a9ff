python -m pytest tests/test_gpu_parity.py -q -x -k "fused_redistribution or ttmc" > gpurun_out/t21.log 2>&1; echo "t rc=$?"; tail -2 gpurun_out/t21.log
PUSH_AB_ONLY=C5:4 timeout 900 python tools/push_ab.py 2>&1 | tail -1
