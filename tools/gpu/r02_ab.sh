# A/B runs of bench.py: each line "name|ENV=... |bench args"; stage times per run
python -m paper_2407_20692_b200.build
while IFS='|' read -r name envs args; do
  [ -z "$name" ] && continue
  env $envs timeout 240 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $args > gpurun_out/r02_ab_$name.json 2> gpurun_out/r02_ab_$name.err
  python -c "import json; d=json.loads(open('gpurun_out/r02_ab_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['value']), {k: round(v, 2) for k, v in d['stages_ms_per_step'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r02_ab_$name.err
done < ${AB:-tools/gpu/ab.txt}
