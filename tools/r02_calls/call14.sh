# full-size C5: discard A/B against the round-1 tree; corrected ncu line profiles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sum
one() { (cd $1 && timeout 900 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
one ab/r1tree C5 0 --steps 3 --warmup 3
one . C5 0 --no-probe --steps 3 --warmup 3
one . C5 0 --no-probe --steps 3 --warmup 3 --lib ab/nodiscard.so
done
cap() {  # name args regex instances
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$3 -s 3 -c 1 -o /tmp/prof_$1 \
    python bench.py $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-probe > /tmp/ncu_$1.log 2>&1; echo "$1 rc=$?"
  python tools/ncu_lines.py /tmp/prof_$1.ncu-rep paper_2011_01112_b200/libicsched.so x 60 > gpurun_out/sum/$1_lines.txt 2>&1
  rm -f /tmp/prof_$1.ncu-rep
}
cap C5 "--config C5 --instances 400000" ic_dp_kernel 400000
cap C2 "--config C2" ic_solo_kernel 100000
cap C3d01 "--config C3 --delta-micro 100000 --instances 200000" ic_solo_kernel 200000
cap C4 "--config C4" ic_dp_kernel 10000
