# 32-bit q division A/B; C4 ncu summary of the final in-place kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sum
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t10.log 2>&1; tail -2 gpurun_out/t10.log
one() { (cd $1 && timeout 600 python bench.py --config $2 --instances ${3:-0} --no-cpu-baseline --no-e2e ${@:4} 2>/dev/null) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 ${*:4}', round(d['value']), round(d['ms_per_step'],3), d.get('result_hash'))" 2>/dev/null || echo "$1 $2 FAILED"; }
for rep in 1 2; do
for l in "" "--lib ab/olddiv.so"; do
one . C2 0 --no-probe $l
one . C2 0 --no-probe --delta-micro 100000 $l
one . C3 0 --no-probe --delta-micro 100000 $l
one . C5 2000000 --no-probe $l
done
done
cap() {  # dir name args regex instances kernel-substring
  (cd $1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:$4 -s 3 -c 1 -o /tmp/prof_$2 \
    python bench.py $3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ncu_$2.log 2>&1; echo "$2 rc=$?")
  python tools/ncu_summary.py /tmp/prof_$2.ncu-rep $2 $5 --round r02 > gpurun_out/sum/$2.json 2>&1
  python tools/ncu_lines.py /tmp/prof_$2.ncu-rep $1/paper_2011_01112_b200/libicsched.so $6 60 > gpurun_out/sum/$2_lines.txt 2>&1
  rm -f /tmp/prof_$2.ncu-rep
}
cap . C4 "--config C4 --no-probe" ic_dp_kernel 10000 ic_dp_kernelILi15
