# Round-2 final measurement: every bench line, the C5 launch list, ncu summaries of the final kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sum
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
bash tools/r02_lines.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-probe > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
cap() {  # name args regex instances kernel-substring
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$3 -s 3 -c 1 -o /tmp/prof_$1 \
    python bench.py $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-probe > /tmp/ncu_$1.log 2>&1; echo "$1 rc=$?"
  python tools/ncu_summary.py /tmp/prof_$1.ncu-rep $1 $4 --round r02 > gpurun_out/sum/$1.json 2>&1
  python tools/ncu_lines.py /tmp/prof_$1.ncu-rep paper_2011_01112_b200/libicsched.so $5 60 > gpurun_out/sum/$1_lines.txt 2>&1
  rm -f /tmp/prof_$1.ncu-rep
}
cap C5 "--config C5 --instances 400000" ic_dp_kernel 400000 ic_dp_kernelILi4
cap C3 "--config C3 --instances 200000" ic_dp_kernel 200000 ic_dp_kernelILi4
cap C2 "--config C2" ic_solo_kernel 100000 ic_solo_kernel
cap C3d01 "--config C3 --delta-micro 100000 --instances 200000" ic_solo_kernel 200000 ic_solo_kernel
cap C4 "--config C4" ic_dp_kernel 10000 ic_dp_kernelILi15
cap reassign_C3 "--op reassign --config C3 --instances 200000" reassign_kernel 200000 reassign
ls -la gpurun_out/sum
