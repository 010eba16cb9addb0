# three-rows-per-load backtrack in the solo kernel (short option lists): parity + A/B
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_sim.py -m gpu -q -x > gpurun_out/t26.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t26.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k C2 > gpurun_out/t26b.log 2>&1; echo "fullsize C2 rc=$?"; tail -1 gpurun_out/t26b.log
one() { (cd $1 && timeout 900 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
for l in "" "--lib ab/prev.so"; do
one . C2 0 --no-probe $l
one . C2 0 --no-probe --delta-micro 100000 $l
one . C1 1000000 --no-probe $l
done
done
