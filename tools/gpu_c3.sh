mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py -m gpu -x -q > gpurun_out/pytest_build.log 2>&1; echo pytest=$? >> gpurun_out/pytest_build.log
timeout 900 python tools/exp_build.py c2 c4 > gpurun_out/build_c2c4.log 2>&1
