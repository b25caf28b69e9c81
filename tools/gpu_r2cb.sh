# r2cb: flat query grid for binned-eligible indexes, c3 at 8 cells per leaf side: c3 and c4 on both paths, launch list, binned/parity/build/c3-full tests
mkdir -p gpurun_out/r2cb
timeout 900 python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2cb/c3.log 2>&1
timeout 900 python tools/exp_binned.py c4 2e8 0 > gpurun_out/r2cb/c4.log 2>&1
timeout 900 python tools/exp_binned.py c2 1e8 0 > gpurun_out/r2cb/c2.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py tests/test_gpu_build.py tests/test_gpu_c3_full.py -x -q > gpurun_out/r2cb/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2cb/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" --csv --log-file gpurun_out/r2cb/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2cb/ncu.log 2>&1
