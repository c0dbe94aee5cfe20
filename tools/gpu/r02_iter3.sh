# iteration: build; named GPU tests (per-test timeout); default + v-major benches (stage times)
python -m paper_2407_20692_b200.build
timeout ${TT:-900} python -m pytest ${TESTS} -q -rf -x --timeout=240 > gpurun_out/r02_it_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_it_tests.log
tail -4 gpurun_out/r02_it_tests.log
for o in ${ORDERS:-ublocked vmajor}; do
  timeout 240 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --gamma-order $o > gpurun_out/r02_it_bench_$o.json 2> gpurun_out/r02_it_bench_$o.err
  python -c "import json; d=json.loads(open('gpurun_out/r02_it_bench_$o.json').read().strip().splitlines()[-1]); print('$o', round(d['value']), {k: round(v, 2) for k, v in d['stages_ms_per_step'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r02_it_bench_$o.err
done
