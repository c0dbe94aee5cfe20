python -m paper_2407_20692_b200.build
timeout 900 python -m pytest tests/test_gpu_vmajor.py -q -x > gpurun_out/r02_iter_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_iter_tests.log
tail -3 gpurun_out/r02_iter_tests.log
PROBES="${PROBES:-0 16}" bash tools/gpu/r02_probe.sh
