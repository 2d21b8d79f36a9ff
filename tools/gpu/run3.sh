python -m pytest tests/test_gpu_parity.py -q -k "gemm" > gpurun_out/gemm_tests.log 2>&1; echo "gemm tests rc=$?"
tail -5 gpurun_out/gemm_tests.log
timeout 900 python tools/gemm_chain_check.py --out gpurun_out/gemm_chain.jsonl > gpurun_out/gemm.log 2>&1; echo "gemm rc=$?"
tail -4 gpurun_out/gemm.log
timeout 600 python tools/sanitize_small.py > gpurun_out/san_plain.log 2>&1; echo "san plain rc=$?"
tail -3 gpurun_out/san_plain.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check full --print-limit 50 python tools/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -30 gpurun_out/san_memcheck.log
