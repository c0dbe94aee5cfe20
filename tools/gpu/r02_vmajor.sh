# v-major window stage 1: parity tests, then bench A/B against the u-blocked TMA stage 1
python -m paper_2407_20692_b200.build
timeout 900 python -m pytest tests/test_gpu_vmajor.py -q -rf -x > gpurun_out/r02_vmajor_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_vmajor_tests.log
tail -5 gpurun_out/r02_vmajor_tests.log
for o in vmajor ublocked vmajor; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --gamma-order $o > gpurun_out/r02_bench_$o.json 2> gpurun_out/r02_bench_$o.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/r02_bench_$o.json').read().strip().splitlines()[-1]); print('$o', d['value'], d['stages_ms_per_step'], d['clocks']['sm_mhz'])"
done
