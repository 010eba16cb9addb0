# decision L2 policy A/B at full size (discard / no discard / evict_last stores), DRAM bytes per variant
cd $GRAFT_REPO_ROOT
one() { (cd $1 && timeout 900 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
for l in "" "--lib ab/nodiscard.so" "--lib ab/keep.so" "--lib ab/keepdisc.so"; do
one . C5 0 --no-probe --steps 3 --warmup 3 $l
done
done
for l in "" "--lib ab/nodiscard.so" "--lib ab/keep.so" "--lib ab/keepdisc.so"; do
one . C2 0 --no-probe $l
one . C3 0 --no-probe --delta-micro 100000 $l
done
for l in "" "--lib ab/nodiscard.so" "--lib ab/keep.so" "--lib ab/keepdisc.so"; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ic_ -s 3 -c 1 --csv \
    python bench.py --config C5 --instances 400000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-probe $l 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v L="$l" '{print L, $(NF-2), $NF}'
done
