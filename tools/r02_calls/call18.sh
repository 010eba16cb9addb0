# ws-kernel discard compiled out: parity subset, C5 full-size A/B against the no-discard build
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/t18.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t18.log
one() { (cd $1 && timeout 900 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
one . C5 0 --no-probe --steps 3 --warmup 3
one . C5 0 --no-probe --steps 3 --warmup 3 --lib ab/keep.so
one . C5 0 --no-probe --steps 3 --warmup 3 --lib ab/wsdisc.so
one . C3 0 --no-probe
one . C3 0 --no-probe --lib ab/keep.so
done
