# perf A/B on one GPU: parity first, then the bench configs (optionally with env overrides)
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x 2>&1 | tail -3
b() { timeout 600 python bench.py --config $1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['roofline']['frac'],4), round(d['ms_per_step'],3))"; }
for c in ${CONFIGS:-C5 C3 C2 C4}; do b $c; done
