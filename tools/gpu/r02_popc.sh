set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --variant popc --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_popc.json 2> gpurun_out/r02_bench_popc.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_base.json 2> gpurun_out/r02_bench_base.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_popc -c 1 -o gpurun_out/r02_popc python bench.py --variant popc --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_popc.log 2>&1
ls -la gpurun_out
