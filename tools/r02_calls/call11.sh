# opaque per-kernel row-buffer addresses A/B (ws kernel: C5, C3; solo unaffected)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t11.log 2>&1; tail -2 gpurun_out/t11.log
one() { (cd $1 && timeout 600 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2 3; do
for l in "" "--lib ab/head2.so"; do
one . C5 2000000 --no-probe $l
one . C3 0 --no-probe $l
done
done
