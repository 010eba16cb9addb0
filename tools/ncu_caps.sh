#!/bin/bash
# ncu --set full captures of the solve kernels (one GPU; under gpurun).  Usage:
#   bash tools/ncu_caps.sh NAME "bench args" KERNEL_REGEX [NAME "args" REGEX ...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
while [ $# -ge 3 ]; do
  name=$1; args=$2; rx=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -s 3 -c 1 -o gpurun_out/prof_$name \
    python bench.py $args --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-probe > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"; tail -1 gpurun_out/ncu_$name.log | cut -c1-200
done
