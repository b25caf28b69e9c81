# r2z: binned histogram from res (dedicated kernel), hist tests, c3/c5 hist timing
mkdir -p gpurun_out/r2z
timeout 1200 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py -x -q > gpurun_out/r2z/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2z/pytest.log
EXPV_HIST=1 timeout 900 python tools/exp_variants.py c3 1e9 binned 0 > gpurun_out/r2z/c3_hist.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"binned_hist|binned_query|widen" --csv --log-file gpurun_out/r2z/launches_hist.csv \
  env EXPV_HIST=1 python tools/exp_variants.py c3 1e9 binned 0 > gpurun_out/r2z/ncu.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --no-cpu --no-e2e --check-points 2000000 > gpurun_out/r2z/c5.log 2>&1
