#!/bin/bash
# End-of-session evidence on one box (run under gpurun): GPU test suite,
# smoke, the headline bench line, then the secondary lines (tools/lines_job.sh).
set -u
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/final/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/final/headline.json 2> gpurun_out/final/headline.log; echo "headline rc=$?"
python tools/stress_launch_ahead.py tiny-shared 100 > gpurun_out/final/stress.log 2>&1; echo "stress rc=$?"; tail -1 gpurun_out/final/stress.log
bash tools/lines_job.sh
