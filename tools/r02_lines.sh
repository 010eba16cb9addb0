#!/bin/bash
# Round-2 measurement set (under gpurun): bench lines for every configuration and operation,
# written to gpurun_out/bench_r02_<name>.json (copied to profiles/ afterwards).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_r02_$name.json 2> gpurun_out/bench_r02_$name.err;
        echo "$name rc=$? $(tail -c 300 gpurun_out/bench_r02_$name.json | tr -d '\n' | cut -c1-160)"; }
run C5_default
run C1 --config C1
run C1_1M --config C1 --instances 1000000 --no-cpu-baseline
run C2 --config C2
run C3 --config C3
run C4 --config C4
run C2_delta01 --config C2 --delta-micro 100000 --no-cpu-baseline
run C3_delta01 --config C3 --delta-micro 100000 --no-cpu-baseline
run C4_delta01 --config C4 --delta-micro 100000 --no-cpu-baseline
run reassign_C2 --op reassign --config C2
run reassign_C3 --op reassign --config C3
run replan_C2 --op replan --config C2 --delta-micro 100000
run replan_C3 --op replan --config C3 --delta-micro 100000 --instances 200000
run replan_C3_time --op replan --config C3 --delta-micro 100000 --instances 200000 --tune axis=1
run simulate --op simulate
run reference_C5 --impl reference --steps 3 --warmup 3
