cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
one() { (cd $1 && timeout 600 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e --no-probe ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
for t in ab/r1tree ab/t_8508c75 ab/t_7340026 ab/t_4b7fd3d .; do one $t C5 2000000; done
done
for rep in 1 2; do
one . C3 0 --delta-micro 100000
one . C3 0 --delta-micro 100000 --tune packed_options=2
one . C2 0 --delta-micro 100000
one . C2 0 --delta-micro 100000 --tune packed_options=2
one . C4 0
one . C4 0 --tune dp_warps=15
done
