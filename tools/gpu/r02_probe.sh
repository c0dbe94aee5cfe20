# KB5w timing probes (wrong values): CPI_S1W_PROBE=1 -> no Gamma TMA loads (entries only)
python -m paper_2407_20692_b200.build
for p in ${PROBES:-0 1 0}; do
  CPI_S1W_PROBE=$p timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --gamma-order vmajor > gpurun_out/r02_probe_$p.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/r02_probe_$p.json').read().strip().splitlines()[-1]); print('probe $p', d['stages_ms_per_step']['refocus_stage1'])"
done
