# r2bs: grouped sampling (4 consecutive points per 256-point stratum): binned tests, launch list
mkdir -p gpurun_out/r2bs
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2bs/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bs/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" --csv --log-file gpurun_out/r2bs/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bs/ncu.log 2>&1
tail -3 gpurun_out/r2bs/ncu.log > gpurun_out/r2bs/c3.log
