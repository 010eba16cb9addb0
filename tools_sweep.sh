#!/bin/bash
# variant sweep (scratch): config, env settings
run() { env $2 python bench.py --config $1 $3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    r=d['roofline']; k=d['kernel']; print('value %.3e frac %.3f kern_ms %.3f' % (d['value'], r['frac'], r['kernel_ms']), 'nw', (k['threads_per_cta']//32)-1, 'ctas', k['ctas_per_sm'], 'smem', k['smem_bytes'], 'decsmem', k['decisions_in_smem'])"; }
for env in "" "IC_SCHED_NW=2" "IC_SCHED_DEC=global1" "IC_SCHED_DEC=smem"; do echo "== C2 $env"; run C2 "$env" ""; done
for env in "" "IC_SCHED_NW=2" "IC_SCHED_NW=1" "IC_SCHED_NW=8"; do echo "== C3 $env"; run C3 "$env" "--instances 200000"; done
for env in "" "IC_SCHED_NW=8"; do echo "== C4 $env"; run C4 "$env" "--instances 2000"; done
echo "== C1"; run C1 "" "--instances 1000000"
