python -m paper_2407_20692_b200.build
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage1_w_kernel -c 1 -o gpurun_out/r02_stage1w_b python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_stage1w_b.log 2>&1
echo "ncu rc=$?"
