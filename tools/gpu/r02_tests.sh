# round-2 GPU run: the whole -m gpu suite (log in gpurun_out/), then smoke()
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2407_20692_b200.build
timeout 3000 python -m pytest tests -m gpu -q -rf --durations=15 ${PYTEST_ARGS} > gpurun_out/r02_gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02_smoke.log
tail -30 gpurun_out/r02_gpu_tests.log
