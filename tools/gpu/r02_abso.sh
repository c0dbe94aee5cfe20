# A/B of prebuilt library variants (abvar/<name>.so, built here with different sources or flags):
# optional parity tests on the first variant, then bench.py runs alternating over the variants.
export CPI_NO_BUILD=1
L=paper_2407_20692_b200/libcpi.so
if [ -n "$TESTS" ]; then
  cp abvar/${VARS%% *}.so $L
  timeout ${TT:-900} python -m pytest $TESTS -q -rf -x --timeout=300 > gpurun_out/r02_abso_tests.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/r02_abso_tests.log
  tail -3 gpurun_out/r02_abso_tests.log
fi
for rep in $(seq ${REPS:-2}); do
  for v in $VARS; do
    cp abvar/$v.so $L
    timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $ARGS > gpurun_out/r02_abso_$v.json 2> gpurun_out/r02_abso_$v.err
    python -c "import json; d=json.loads(open('gpurun_out/r02_abso_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), {k: round(v, 2) for k, v in d['stages_ms_per_step'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r02_abso_$v.err
  done
done
