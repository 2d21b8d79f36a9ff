timeout 600 python tools/sanitize_small.py > gpurun_out/san_plain.log 2>&1; echo "san plain rc=$?"
tail -3 gpurun_out/san_plain.log
python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/gputests.log 2>&1; echo "gpu rc=$?"
tail -45 gpurun_out/gputests.log
