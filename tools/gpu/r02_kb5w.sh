# KB5w iteration: build, v-major parity tests, v-major bench (stage times), then timing probes
python -m paper_2407_20692_b200.build
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_vmajor.py} -q -rf -x > gpurun_out/r02_kb5w_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_kb5w_tests.log
tail -4 gpurun_out/r02_kb5w_tests.log
for p in ${PROBES:-0 16 0}; do
  CPI_S1W_PROBE=$p timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --gamma-order vmajor > gpurun_out/r02_kb5w_probe_$p.json 2> gpurun_out/r02_kb5w_probe_$p.err
  python -c "import json; d=json.loads(open('gpurun_out/r02_kb5w_probe_$p.json').read().strip().splitlines()[-1]); print('probe $p', d['stages_ms_per_step'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r02_kb5w_probe_$p.err
done
