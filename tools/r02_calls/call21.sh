# plain (unhinted) stores for re-plan state decisions: replan lines and C5 against the previous build
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "replan or departures or decision or variant" > gpurun_out/t21.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t21.log
one() { (cd $1 && timeout 900 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'), d.get('speedup_vs_full_solve'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
for l in "" "--lib ab/prev.so"; do
one . C2 0 --op replan --delta-micro 100000 $l
one . C3 200000 --op replan --delta-micro 100000 $l
one . C5 0 --no-probe --steps 3 --warmup 3 $l
done
done
