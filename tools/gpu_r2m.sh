# r2m: resolve double batches + scatter per16: tests, c3 paths, full ncu capture of scatter + query
mkdir -p gpurun_out/r2m
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binned.py tests/test_gpu_margin.py -x -q > gpurun_out/r2m/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2m/pytest.log
timeout 1200 python tools/exp_binned.py c3 1e9 64e6 > gpurun_out/r2m/c3.log 2>&1; echo rc=$? >> gpurun_out/r2m/c3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bin_scatter|binned_query|resolve_kernel" -c 3 \
  -o gpurun_out/r2m/prof python tools/exp_binned.py c3 1e9 64e6 > gpurun_out/r2m/ncu_full.log 2>&1; echo rc=$? >> gpurun_out/r2m/ncu_full.log
