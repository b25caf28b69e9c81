# r2az: slot staging with one multiply-add per source address and per-lane constant destinations: binned + parity tests, A/B c3/c4
mkdir -p gpurun_out/r2az
timeout 900 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py -x -q > gpurun_out/r2az/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2az/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2az/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2az/ab_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"binned_query" --csv --log-file gpurun_out/r2az/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2az/ncu.log 2>&1
