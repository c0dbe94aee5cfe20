# ncu --set full of the KB5w stage 1 (v-major bench step) + launch list of the v-major step
python -m paper_2407_20692_b200.build
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage1_w_kernel -c 1 -o gpurun_out/r02_stage1w python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_stage1w.log 2>&1
echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_vm.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_launch_vm.log 2>&1
echo "launches rc=$?"
