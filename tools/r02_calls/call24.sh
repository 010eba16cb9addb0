# final build: GPU suite + smoke; refreshed lines for the configurations the K = 5 solo kernel serves
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sum
timeout 1500 python -m pytest tests -m gpu -q -ra > gpurun_out/gputest_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
cap() {  # name args regex instances
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$3 -s 3 -c 1 -o /tmp/prof_$1 \
    python bench.py $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-probe > /tmp/ncu_$1.log 2>&1; echo "$1 rc=$?"
  python tools/ncu_summary.py /tmp/prof_$1.ncu-rep $1 $4 --round r02 > gpurun_out/sum/$1.json 2>&1
  python tools/ncu_lines.py /tmp/prof_$1.ncu-rep paper_2011_01112_b200/libicsched.so x 60 > gpurun_out/sum/$1_lines.txt 2>&1
  rm -f /tmp/prof_$1.ncu-rep
}
cap C2 "--config C2" ic_solo_kernel 100000
cap C2d01 "--config C2 --delta-micro 100000" ic_solo_kernel 100000
for n in C2 C2d01; do python -c "import json;json.load(open('gpurun_out/sum/$n.json'))" && cp gpurun_out/sum/$n.json profiles/ncu_${n}_summary.json; done
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_r02_$name.json 2> gpurun_out/bench_r02_$name.err;
        echo "$name rc=$? $(tail -c 300 gpurun_out/bench_r02_$name.json | tr -d '\n' | cut -c1-100)"; }
run C1 --config C1
run C1_1M --config C1 --instances 1000000 --no-cpu-baseline
run C2 --config C2
run C2_delta01 --config C2 --delta-micro 100000 --no-cpu-baseline
run replan_C2 --op replan --config C2 --delta-micro 100000
run reassign_C2 --op reassign --config C2
