# C4 chunk size A/B (15-warp kernel); ncu line profiles of the solo kernel (C2, C3 at Delta=0.1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sum
one() { (cd $1 && timeout 600 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
one . C4 0 --no-probe
one . C4 0 --no-probe --lib ab/ch16.so
done
cap() {  # dir name args regex instances kernel-substring
  (cd $1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:$4 -s 3 -c 1 -o /tmp/prof_$2 \
    python bench.py $3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu_$2.log 2>&1; echo "$2 rc=$?")
  python tools/ncu_summary.py /tmp/prof_$2.ncu-rep $2 $5 --round r02 > gpurun_out/sum/$2.json 2>&1
  python tools/ncu_lines.py /tmp/prof_$2.ncu-rep $1/paper_2011_01112_b200/libicsched.so $6 90 > gpurun_out/sum/$2_lines.txt 2>&1
  rm -f /tmp/prof_$2.ncu-rep
}
cap . C2 "--config C2 --no-probe" ic_solo_kernel 100000 ic_solo_kernel
cap . C3d01 "--config C3 --delta-micro 100000 --instances 200000 --no-probe" ic_solo_kernel 200000 ic_solo_kernel
cap . C5 "--config C5 --instances 400000 --no-probe" ic_dp_kernel 400000 ic_dp_kernelILi4
ls -la gpurun_out/sum
