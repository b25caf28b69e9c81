# r2bn: scatter (tile-level key, whole-chunk count path) + unbin (ballot run lookup): binned + parity tests, c3/c4 A/B against the r2be code, launch list
mkdir -p gpurun_out/r2bn
timeout 900 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py -x -q > gpurun_out/r2bn/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bn/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bn/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bn/ab_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" --csv --log-file gpurun_out/r2bn/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bn/ncu.log 2>&1
