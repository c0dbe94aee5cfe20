python -m paper_2407_20692_b200.build
timeout ${TT:-900} python -m pytest ${TESTS} -q -rf -x --timeout=240 > gpurun_out/r02_it_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_it_tests.log
tail -4 gpurun_out/r02_it_tests.log
AB=${AB} bash tools/gpu/r02_ab.sh
