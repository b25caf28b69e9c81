# r2bk: scatter with an fp32 tile key, whole-chunk / no-overflow fast paths; unbin run lookup by ballot + one shuffle: binned tests, A/B, launch list
mkdir -p gpurun_out/r2bk
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2bk/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bk/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bk/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bk/ab_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" --csv --log-file gpurun_out/r2bk/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bk/ncu.log 2>&1
