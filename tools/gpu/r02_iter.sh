# iteration: build, the named GPU tests, then the v-major bench (stage times)
python -m paper_2407_20692_b200.build
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_vmajor.py} -q -rf > gpurun_out/r02_iter_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_iter_tests.log
tail -8 gpurun_out/r02_iter_tests.log
for o in ${ORDERS:-vmajor}; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --gamma-order $o > gpurun_out/r02_bench_$o.json 2> gpurun_out/r02_bench_$o.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/r02_bench_$o.json').read().strip().splitlines()[-1]); print('$o', d['value'], d['stages_ms_per_step'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/r02_bench_$o.err
done
