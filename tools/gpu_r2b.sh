# round 2: binned path parity + c3/c4/c2 bench lines + c3 launch list
mkdir -p gpurun_out/r2b
timeout 1200 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py -x -q > gpurun_out/r2b/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2b/pytest.log
timeout 1500 python bench.py --config c3 --points 1000000000 --no-cpu --no-e2e --steps 5 > gpurun_out/r2b/c3_1B.log 2>&1; echo rc=$? >> gpurun_out/r2b/c3_1B.log
timeout 900 python bench.py --config c4 --no-cpu --no-e2e --steps 5 > gpurun_out/r2b/c4.log 2>&1; echo rc=$? >> gpurun_out/r2b/c4.log
timeout 900 python bench.py --config c2 --no-cpu --no-e2e --steps 5 > gpurun_out/r2b/c2.log 2>&1; echo rc=$? >> gpurun_out/r2b/c2.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"bin_|binned|unbin" --csv --log-file gpurun_out/r2b/launches_c3.csv \
  python bench.py --config c3 --points 1000000000 --no-cpu --no-e2e --steps 1 --warmup 0 > gpurun_out/r2b/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/r2b/ncu_c3.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"bin_|binned|unbin" --csv --log-file gpurun_out/r2b/launches_c4.csv \
  python bench.py --config c4 --no-cpu --no-e2e --steps 1 --warmup 0 > gpurun_out/r2b/ncu_c4.log 2>&1; echo rc=$? >> gpurun_out/r2b/ncu_c4.log
