# r2s: copy/fronts microbenchmark + per-lane staging (tests, c3 binned/stream)
mkdir -p gpurun_out/r2s
./tools/exp_copy.bin > gpurun_out/r2s/copy.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binned.py tests/test_gpu_margin.py tests/test_gpu_build.py -x -q > gpurun_out/r2s/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2s/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|stream_kernel|resolve_kernel" --csv --log-file gpurun_out/r2s/launches_c3.csv \
  python tools/exp_binned.py c3 1e9 64e6 > gpurun_out/r2s/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/r2s/ncu_c3.log
timeout 1200 python tools/exp_binned.py c3 1e9 16e6 64e6 > gpurun_out/r2s/c3.log 2>&1; echo rc=$? >> gpurun_out/r2s/c3.log
