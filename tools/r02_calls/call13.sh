# backtrack prefetch A/B, hybrid state path parity + replan line, full-size C5 vs round-1 tree, C5 launch list
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t13.log 2>&1; tail -2 gpurun_out/t13.log
one() { (cd $1 && timeout 900 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'), d.get('speedup_vs_full_solve'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
for l in "" "--lib ab/head3.so"; do
one . C2 0 --no-probe $l
one . C2 0 --no-probe --delta-micro 100000 $l
one . C3 0 --no-probe --delta-micro 100000 $l
done
done
one . C3 200000 --op replan --delta-micro 100000
one . C2 0 --op replan --delta-micro 100000
for rep in 1 2; do
one ab/r1tree C5 0 --steps 4 --warmup 3
one . C5 0 --no-probe --steps 4 --warmup 3
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C5sub.csv \
  python bench.py --instances 400000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-probe > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
