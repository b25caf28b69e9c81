# r2u: smem-attribute fix; binned tests; c3 + c4 path timings
mkdir -p gpurun_out/r2u
timeout 1500 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py tests/test_gpu_margin.py -x -q > gpurun_out/r2u/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2u/pytest.log
timeout 1200 python tools/exp_binned.py c3 1e9 32e6 64e6 128e6 > gpurun_out/r2u/c3.log 2>&1; echo rc=$? >> gpurun_out/r2u/c3.log
timeout 900 python tools/exp_binned.py c4 2e8 8e6 32e6 128e6 > gpurun_out/r2u/c4.log 2>&1; echo rc=$? >> gpurun_out/r2u/c4.log
timeout 900 python tools/exp_binned.py c2 1e8 32e6 128e6 > gpurun_out/r2u/c2.log 2>&1; echo rc=$? >> gpurun_out/r2u/c2.log
