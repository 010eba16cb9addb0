# env-knob sweep on one box: "ENV=val ... :config[:instances]" entries
mkdir -p gpurun_out
for spec in "$@"; do
  envs=${spec%%:*}; rest=${spec#*:}; c=${rest%%:*}; n=${rest#*:}; [ "$n" = "$rest" ] && n=0
  r=$(env $envs timeout 600 python bench.py --config $c --instances $n --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4), round(d['ms_per_step'],3))")
  echo "$spec -> $r"
done
