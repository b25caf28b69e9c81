mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py -m gpu -x -q > gpurun_out/pytest_build.log 2>&1; echo pytest=$? >> gpurun_out/pytest_build.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_parity.log 2>&1; echo pytest=$? >> gpurun_out/pytest_parity.log
timeout 300 python tools/exp_sweep.py 0 > gpurun_out/sweep_build.log 2>&1
