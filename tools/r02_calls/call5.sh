# round-2 A/B: parity of the working tree, then bench lines vs the round-1 tree
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sanitizer.py -m gpu -x -q > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
one() { (cd $1 && timeout 600 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
one ab/r1tree C5 2000000
one . C5 2000000 --no-probe
one ab/r1tree C3 0
one . C3 0 --no-probe
one . C3 0 --no-probe --delta-micro 100000
one . C3 0 --no-probe --delta-micro 100000 --tune packed_options=2
one . C2 0 --no-probe --delta-micro 100000
one . C2 0 --no-probe
one ab/r1tree C4 0
one . C4 0 --no-probe
one . C4 0 --no-probe --tune dp_warps=15
done
