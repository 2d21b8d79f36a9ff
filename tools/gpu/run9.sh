timeout 600 python tools/sanitize_small.py > gpurun_out/san_plain.log 2>&1; echo "san plain rc=$?"
tail -2 gpurun_out/san_plain.log
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu rc=$?"
tail -5 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
