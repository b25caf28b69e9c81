# r2ah: sampled single-pass binning -- binned GPU tests, A/B against the counting pass (c3, c4), launch list
mkdir -p gpurun_out/r2ah
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2ah/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ah/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 900 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_count.so $V/lib_sample.so $V/lib_count.so $V/lib_sample.so > gpurun_out/r2ah/ab_c3.log 2>&1
timeout 600 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_count.so $V/lib_sample.so > gpurun_out/r2ah/ab_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" --csv --log-file gpurun_out/r2ah/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2ah/ncu.log 2>&1
