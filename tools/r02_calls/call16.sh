# final round-2 check: GPU test suite, smoke, bench lines of the final build, ncu summaries of the ws kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sum
timeout 1500 python -m pytest tests -m gpu -q -ra > gpurun_out/gputest_final.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_r02_$name.json 2> gpurun_out/bench_r02_$name.err;
        echo "$name rc=$? $(tail -c 300 gpurun_out/bench_r02_$name.json | tr -d '\n' | cut -c1-120)"; }
cap() {  # name args regex instances
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$3 -s 3 -c 1 -o /tmp/prof_$1 \
    python bench.py $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-probe > /tmp/ncu_$1.log 2>&1; echo "$1 rc=$?"
  python tools/ncu_summary.py /tmp/prof_$1.ncu-rep $1 $4 --round r02 > gpurun_out/sum/$1.json 2>&1
  python tools/ncu_lines.py /tmp/prof_$1.ncu-rep paper_2011_01112_b200/libicsched.so x 60 > gpurun_out/sum/$1_lines.txt 2>&1
  rm -f /tmp/prof_$1.ncu-rep
}
cap C5 "--config C5 --instances 400000" ic_dp_kernel 400000
cap C3 "--config C3 --instances 200000" ic_dp_kernel 200000
cap C4 "--config C4" ic_dp_kernel 10000
cp profiles/ncu_C5_summary.json /tmp/ 2>/dev/null; for n in C5 C3 C4; do python -c "import json;json.load(open('gpurun_out/sum/$n.json'))" && cp gpurun_out/sum/$n.json profiles/ncu_${n}_summary.json; done
run C5_default
run C3 --config C3
run C4 --config C4
run C2 --config C2
run C2_delta01 --config C2 --delta-micro 100000 --no-cpu-baseline
run C3_delta01 --config C3 --delta-micro 100000 --no-cpu-baseline
run replan_C2 --op replan --config C2 --delta-micro 100000
run replan_C3 --op replan --config C3 --delta-micro 100000 --instances 200000
run replan_C3_time --op replan --config C3 --delta-micro 100000 --instances 200000 --tune axis=1
