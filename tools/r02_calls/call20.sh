# final bench lines of the final build (every configuration and operation), C5 launch list
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
bash tools/r02_lines.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C5sub.csv \
  python bench.py --instances 400000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-probe > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
