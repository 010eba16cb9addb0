#!/bin/bash
# A/B of two source trees on one box: ab/<tree>/ (a `git archive` of an older revision with its
# own in-tree build) against the working tree, alternating, same configs.
# usage: TREE=r1tree bash tools/ab_tree.sh "C5:2000000 C3 C3:0:100000"   (config[:instances[:delta]])
mkdir -p gpurun_out
root=$(pwd)
run() {  # $1 = label, $2 = config spec, $3 = directory
  local spec=$2 c n dm
  IFS=: read -r c n dm <<< "$spec"
  (cd "$3" && timeout 600 python bench.py --config $c --instances ${n:-0} ${dm:+--delta-micro $dm} --no-cpu-baseline --no-e2e $EXTRA 2>/dev/null) | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['roofline']['frac'],4), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"
}
for rep in 1 2; do
  for c in $1; do
    run ${TREE:-r1tree} $c "$root/ab/${TREE:-r1tree}"
    run new $c "$root"
  done
done
