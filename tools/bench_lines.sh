#!/bin/bash
# Several short bench lines in one GPU session (A/B of tunings / configs).  Each argument is
# one quoted set of bench.py flags; a line of summary per run goes to gpurun_out/lines.txt and
# the full JSON to gpurun_out/line_<i>.json.   bash tools/bench_lines.sh "--config C2" "--config C2 --tune kernel=1"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
i=0
for a in "$@"; do
  i=$((i+1))
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $a > gpurun_out/line_$i.json 2> gpurun_out/line_$i.err
  python - "$i" "$a" <<'PY' >> gpurun_out/lines.txt
import json, sys
i, a = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/line_{i}.json").read().strip().splitlines()[-1])
    r = d.get("roofline", {})
    print(f"{a:50s} value={d['value']:.4g} frac={r.get('frac', 0):.3f} kern_ms={r.get('kernel_ms', 0):.3f} "
          f"hash={d.get('result_hash')} clk={d.get('clocks', {}).get('sm_mhz')} kernel={d.get('kernel', {})}")
except Exception as e:
    print(f"{a:50s} FAILED {e}: " + open(f"gpurun_out/line_{i}.err").read()[-500:].replace(chr(10), ' | '))
PY
done
cat gpurun_out/lines.txt
