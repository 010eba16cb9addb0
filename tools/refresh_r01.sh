# Round-1 refresh on one B200: parity, smoke, bench lines for every config, C5 ncu captures.
mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5) > gpurun_out/r_pytest.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/r_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_r01_C5_default_${V:-v3}.json 2> gpurun_out/r_c5.err
for c in C3 C4 C2 C1; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_r01_${c}_${V:-v3}.json 2> gpurun_out/r_$c.err; done
for c in C2 C3 C4; do timeout 600 python bench.py --config $c --delta-micro 100000 --no-cpu-baseline --no-e2e > gpurun_out/bench_r01_${c}_delta01_${V:-v3}.json 2>/dev/null; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ic_dp_kernel -s 3 -c 1 -o gpurun_out/prof_r01_C5_${V:-v3} python bench.py --config C5 --instances 400000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_C5sub_${V:-v3}.csv python bench.py --config C5 --instances 400000 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cat gpurun_out/r_pytest.txt gpurun_out/r_smoke.txt
for f in gpurun_out/bench_r01_*_${V:-v3}.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], round(d['roofline']['frac'],4), d.get('e2e',{}).get('value'), d.get('latency'))"; done
