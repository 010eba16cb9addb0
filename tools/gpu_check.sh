#!/bin/bash
# One GPU session: the GPU test suite, then bench lines.  Usage (under gpurun):
#   bash tools/gpu_check.sh [pytest -k expr] [bench args...]
# Logs land in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-}
shift || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
if [ "$K" != "none" ]; then
  timeout 3000 python -m pytest tests -m gpu -q -ra --durations=25 ${K:+-k "$K"} > gpurun_out/gputest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/gputest.log
  tail -5 gpurun_out/gputest.log
fi
if [ $# -gt 0 ]; then
  timeout 1200 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json
fi
