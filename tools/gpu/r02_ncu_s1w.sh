# ncu --set full of one window stage-1 launch (64-plane stack, configs[1] Gamma) + source counters
python -m paper_2407_20692_b200.build
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage1_w_kernel -c 1 -o gpurun_out/r02_s1w \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --gamma-order vmajor > gpurun_out/r02_ncu_s1w.log 2>&1
tail -3 gpurun_out/r02_ncu_s1w.log
