# whole-frame stress with the SYRK GEMM vs the full GEMM (CPI_NO_SYRK=1)
python -m paper_2407_20692_b200.build
CPI_SYRK=1 timeout 900 python tools/full_array.py > gpurun_out/r02_full_array_syrk.json 2> gpurun_out/r02_full_array_syrk.err
timeout 900 python tools/full_array.py > gpurun_out/r02_full_array_nosyrk.json 2> gpurun_out/r02_full_array_nosyrk.err
cat gpurun_out/r02_full_array_syrk.json gpurun_out/r02_full_array_nosyrk.json
tail -3 gpurun_out/r02_full_array_syrk.err
