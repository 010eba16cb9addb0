# solo kernel software pipelining A/B (+ parity)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "solo or hybrid or packed or reward or replan or departures or variant or paper" > gpurun_out/t9.log 2>&1; tail -2 gpurun_out/t9.log
one() { (cd $1 && timeout 600 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
for l in "" "--lib ab/nopipe.so"; do
one . C2 0 --no-probe $l
one . C2 0 --no-probe --delta-micro 100000 $l
one . C3 0 --no-probe --delta-micro 100000 $l
one . C1 1000000 --no-probe $l
done
done
