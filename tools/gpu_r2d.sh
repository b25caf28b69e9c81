mkdir -p gpurun_out/r2d
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2d/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2d/pytest.log
timeout 1200 python tools/exp_binned.py c3 1e9 8e6 32e6 128e6 > gpurun_out/r2d/c3.log 2>&1; echo rc=$? >> gpurun_out/r2d/c3.log
timeout 600 python tools/exp_binned.py c4 2e8 16e6 64e6 256e6 > gpurun_out/r2d/c4.log 2>&1; echo rc=$? >> gpurun_out/r2d/c4.log
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"bin_|binned|unbin" --csv --log-file gpurun_out/r2d/launches_c3.csv \
  python tools/exp_binned.py c3 1e9 32e6 > gpurun_out/r2d/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/r2d/ncu_c3.log
( time timeout 1500 python bench.py ) > gpurun_out/r2d/bench.log 2>&1; echo rc=$? >> gpurun_out/r2d/bench.log
