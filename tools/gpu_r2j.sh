# r2j: double leaf slots + global-cursor scatter: GPU build identity + parity + binned, c3 sweep
mkdir -p gpurun_out/r2j
timeout 1500 python -m pytest tests/test_gpu_build.py tests/test_gpu_parity.py tests/test_gpu_binned.py tests/test_gpu_margin.py tests/test_gpu_approx.py tests/test_gpu_simple.py -x -q > gpurun_out/r2j/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2j/pytest.log
timeout 1800 python tools/exp_c3res.py c3 1e9 0 6.5 > gpurun_out/r2j/c3res.log 2>&1; echo rc=$? >> gpurun_out/r2j/c3res.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|stream_kernel|resolve_kernel" --csv --log-file gpurun_out/r2j/launches_c3.csv \
  python tools/exp_binned.py c3 1e9 128e6 > gpurun_out/r2j/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/r2j/ncu_c3.log
