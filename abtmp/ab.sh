P=paper_2407_20692_b200
export CPI_NO_BUILD=1
cp abtmp/libcpi_new.so $P/libcpi.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -q -m gpu -x -k "refocus or affine or fractional or ublocked or cyclic" 2>&1 | tail -3
for i in 1 2; do
  cp abtmp/libcpi_new.so $P/libcpi.so; timeout 300 python bench.py > gpurun_out/n_$i.json 2>/dev/null
  cp abtmp/libcpi_old.so $P/libcpi.so; timeout 300 python bench.py > gpurun_out/o_$i.json 2>/dev/null
done
cp abtmp/libcpi_new.so $P/libcpi.so
for f in gpurun_out/n_*.json gpurun_out/o_*.json; do python -c "import json,sys;d=json.load(open(sys.argv[1]));s=d['stages_ms_per_step'];print(sys.argv[1],round(d['value']),round(s['gemm'],2),round(s['refocus_stage1'],2),round(s['refocus_stage2'],2),d['clocks']['sm_mhz'])" $f; done
