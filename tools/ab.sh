# A/B on one box: ab/$A.so vs the in-tree library, alternating, same configs.
# usage: A=base bash tools/ab.sh "C3 C2 C5:2000000"
mkdir -p gpurun_out
run() {  # $1 = label, $2 = config[:instances]
  local c=${2%%:*} n=${2#*:}; [ "$n" = "$2" ] && n=0
  timeout 600 python bench.py --config $c --instances $n --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['roofline']['frac'],4), round(d['ms_per_step'],3))"
}
for rep in 1 2; do
  for c in $1; do
    IC_SCHED_LIB=ab/${A:-base}.so run "${A:-base}" $c
    run new $c
  done
done
