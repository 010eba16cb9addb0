mkdir -p gpurun_out
r() { env $1 IC_SCHED_LIB=$2 timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['roofline']['frac'],4), d['kernel']['ctas_per_sm'], d['kernel']['pad_cols'], d['result_hash'])"; }
for rep in 1 2; do
r X=1 ""; r IC_SCHED_PAD=64 ""; r X=1 ab/minb14.so; r IC_SCHED_PAD=64 ab/minb14.so; r X=1 ab/minb16.so; r IC_SCHED_PAD=64 ab/minb16.so
done
