# round-2 measurement: GPU suite, smoke, bench (default + v-major), sharded one-rank bench, launch list, ncu
set -x
python -m paper_2407_20692_b200.build
timeout 3000 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --gamma-order vmajor > gpurun_out/r02_bench_vmajor.json 2> gpurun_out/r02_bench_vmajor.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --sharded --parallel-mode lib > gpurun_out/r02_bench_lib1.json 2> gpurun_out/r02_bench_lib1.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --sharded --parallel-mode lib --no-fused-reduce > gpurun_out/r02_bench_lib1_rs.json 2> gpurun_out/r02_bench_lib1_rs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage1_tma_kernel -s 8 -c 1 -o gpurun_out/r02_stage1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_stage1.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_tc2 -c 1 -o gpurun_out/r02_gemm python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_gemm.log 2>&1
tail -5 gpurun_out/r02_gpu_tests.log; tail -2 gpurun_out/r02_smoke.log
