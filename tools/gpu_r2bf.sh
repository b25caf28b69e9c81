# r2bf: binned histogram with a CTA-persistent 16K-slot table over contiguous answer ranges: hist tests, c5 bench, launch list
mkdir -p gpurun_out/r2bf
timeout 900 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py -x -q -k "hist or Hist" > gpurun_out/r2bf/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bf/pytest.log
timeout 900 python bench.py --config c5 --steps 3 --no-cpu --no-e2e --check-points 2000000 > gpurun_out/r2bf/c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"binned_hist|widen" -c 12 --csv --log-file gpurun_out/r2bf/launches_hist.csv python bench.py --config c5 --steps 1 --warmup 0 --no-cpu --no-e2e --check-points 1000000 > gpurun_out/r2bf/ncu.log 2>&1
