# ncu --set full captures: round-1 tree vs working tree on the C5 slice; C4 (15 DP warps), C2, C3 at Delta=0.1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(cd ab/r1tree && timeout 900 ncu --set full --import-source on --clock-control none -k regex:ic_dp_kernel -s 3 -c 1 -o ../../gpurun_out/prof_r1_C5 \
    python bench.py --config C5 --instances 400000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > ../../gpurun_out/ncu_r1_C5.log 2>&1; echo "r1 rc=$?")
bash tools/ncu_caps.sh C5 "--config C5 --instances 400000" ic_dp_kernel C4 "--config C4" ic_dp_kernel C2 "--config C2" ic_solo_kernel C3d01 "--config C3 --delta-micro 100000 --instances 200000" ic_solo_kernel
ls -la gpurun_out/*.ncu-rep
