# r2n: static-block scatter (no barrier/global atomic), resolve back to inline doubles + L2 tail prefetch
mkdir -p gpurun_out/r2n
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binned.py tests/test_gpu_margin.py -x -q > gpurun_out/r2n/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2n/pytest.log
timeout 1200 python tools/exp_binned.py c3 1e9 32e6 64e6 > gpurun_out/r2n/c3.log 2>&1; echo rc=$? >> gpurun_out/r2n/c3.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|stream_kernel|resolve_kernel" --csv --log-file gpurun_out/r2n/launches_c3.csv \
  python tools/exp_binned.py c3 1e9 64e6 > gpurun_out/r2n/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/r2n/ncu_c3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bin_scatter|binned_query" -c 2 \
  -o gpurun_out/r2n/prof python tools/exp_binned.py c3 1e9 64e6 > gpurun_out/r2n/ncu_full.log 2>&1; echo rc=$? >> gpurun_out/r2n/ncu_full.log
