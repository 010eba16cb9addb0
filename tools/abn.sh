# A/B/n on one box: every ab/<label>.so plus the in-tree library ("new"), alternating.
# usage: LIBS="base split2" bash tools/abn.sh "C5:2000000 C3"
mkdir -p gpurun_out
run() {  # $1 = label, $2 = config[:instances], $3 = library ("" = in-tree)
  local c=${2%%:*} n=${2#*:}; [ "$n" = "$2" ] && n=0
  timeout 600 python bench.py ${3:+--lib $3} --config $c --instances $n --no-cpu-baseline --no-e2e $EXTRA 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['roofline']['frac'],4), round(d['ms_per_step'],3), d.get('result_hash'))"
}
for rep in 1 2; do
  for c in $1; do
    for l in $LIBS; do run $l $c ab/$l.so; done
    run new $c ""
  done
done
