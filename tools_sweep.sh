#!/bin/bash
run() { env $2 python bench.py --config $1 $3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    r=d['roofline']; k=d['kernel']; print('value %.3e frac %.3f kern_ms %.3f' % (d['value'], r['frac'], r['kernel_ms']), 'nw', (k['threads_per_cta']//32)-1, 'ctas', k['ctas_per_sm'], 'smem', k['smem_bytes'], 'decsmem', k['decisions_in_smem'])"; }
for a in "$@"; do cfg=${a%%:*}; env=${a#*:}; [ "$env" = "$a" ] && env=""; inst=""; [ "$cfg" = "C3" ] && inst="--instances 200000"; [ "$cfg" = "C4" ] && inst="--instances 2000"; [ "$cfg" = "C1" ] && inst="--instances 1000000"; echo "== $cfg $env"; run $cfg "$env" "$inst"; done
