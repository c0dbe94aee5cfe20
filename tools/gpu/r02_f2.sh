python -m paper_2407_20692_b200.build
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_fused_reduce.py tests/test_gpu_abi_multi.py} -q -rf -x > gpurun_out/r02_f2_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_f2_tests.log
tail -30 gpurun_out/r02_f2_tests.log
