timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_approx.py -m gpu -x -q > gpurun_out/t22.log 2>&1; echo rc=$? >> gpurun_out/t22.log
timeout 600 python bench.py --hist --no-cpu --no-e2e > gpurun_out/c2_hist32r.log 2>&1
timeout 2400 python bench.py --config c5 --points 1000000000 --hist --no-cpu --no-e2e --steps 3 > gpurun_out/c5_hist32r.log 2>&1; echo rc=$? >> gpurun_out/c5_hist32r.log
