# r2g: new GPU tests (margin scale, full c3, multi-GPU entry) + c3 grid-resolution sweep
mkdir -p gpurun_out/r2g
timeout 1200 python -m pytest tests/test_gpu_margin.py tests/test_gpu_multi.py tests/test_gpu_c3_full.py -x -q > gpurun_out/r2g/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2g/pytest.log
timeout 2400 python tools/exp_c3res.py c3 1e9 0 6.5 9.3 > gpurun_out/r2g/c3res.log 2>&1; echo rc=$? >> gpurun_out/r2g/c3res.log
