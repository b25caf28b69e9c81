# r2ad: scatter with shuffle scan + staged destinations; adapter (rebuilt); c3/c4 timings
mkdir -p gpurun_out/r2ad
timeout 1500 python -m pytest tests/test_cpp_adapter.py tests/test_gpu_binned.py tests/test_gpu_parity.py -x -q > gpurun_out/r2ad/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ad/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"bin_|binned|unbin" --csv --log-file gpurun_out/r2ad/launches_c3.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2ad/ncu.log 2>&1
timeout 900 python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2ad/c3.log 2>&1
timeout 900 python tools/exp_binned.py c4 2e8 0 > gpurun_out/r2ad/c4.log 2>&1
