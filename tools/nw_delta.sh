# DP-warp count for the reward-indexed sweep at the paper's Delta = 0.1 (env-knob sweep)
mkdir -p gpurun_out
r() { env $1 timeout 300 python bench.py --config $2 --delta-micro 100000 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['roofline']['frac'],4), d['kernel']['ctas_per_sm'], d['result_hash'])"; }
for nw in 0 1 2 4; do [ $nw = 0 ] && e=X=1 || e=IC_SCHED_NW=$nw; r $e C3; done
for nw in 0 2 4 8; do [ $nw = 0 ] && e=X=1 || e=IC_SCHED_NW=$nw; r $e C4; done
