# uniform decision-placement flag instead of __isGlobal: GPU suite, C5/C3 against the no-guard build
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -ra > gpurun_out/gputest_final.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
one() { (cd $1 && timeout 900 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
one . C5 0 --no-probe --steps 3 --warmup 3
one . C5 0 --no-probe --steps 3 --warmup 3 --lib ab/keep.so
one . C3 0 --no-probe
one . C3 0 --no-probe --lib ab/keep.so
done
