# round-2 closing measurement (after the KB5w byte-offset entries): GPU suite, smoke, bench (default v-major +
# u-blocked), oracle reference arm, launch list, ncu --set full of the KB5w stage 1 and the FP4 GEMM
set -x
python -m paper_2407_20692_b200.build
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/r02g_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02g_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02g_smoke.log
timeout 900 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --gamma-order ublocked > gpurun_out/r02g_bench_ublocked.json 2> gpurun_out/r02g_bench_ublocked.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02g_bench_reference.json 2> gpurun_out/r02g_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02g_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02g_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage1_w_kernel -c 1 -o gpurun_out/r02g_stage1w python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02g_ncu_stage1w.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_tc2 -s 1 -c 1 -o gpurun_out/r02g_gemm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02g_ncu_gemm.log 2>&1
tail -5 gpurun_out/r02g_gpu_tests.log; tail -2 gpurun_out/r02g_smoke.log
