#!/bin/bash
# Full validation on one B200: GPU test suite, smoke, the default bench line.
set -x
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/val_gputests.log 2>&1; echo "gpu rc=$?"
tail -5 gpurun_out/val_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/val_smoke.log
timeout 600 python bench.py > gpurun_out/val_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/val_bench.log | cut -c1-600
