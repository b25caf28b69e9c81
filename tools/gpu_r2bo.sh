# r2bo: unbin with whole-chunk / no-overflow fast paths and four consecutive points per thread (8-byte index loads, 16-byte id stores), at 2 / 3 / 4 CTAs per SM
mkdir -p gpurun_out/r2bo
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2bo/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bo/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_prev.so $V/lib_ub2.so $V/lib_ub4.so $V/lib_prev.so > gpurun_out/r2bo/ab_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"unbin" --csv --log-file gpurun_out/r2bo/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bo/ncu.log 2>&1
