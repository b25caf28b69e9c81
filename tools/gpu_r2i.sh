# r2i: small-record policy (overflow record instead of split subtrees): GPU build identity +
# parity, then c3 stats/build time/query times at two resolutions
mkdir -p gpurun_out/r2i
timeout 1500 python -m pytest tests/test_gpu_build.py tests/test_gpu_parity.py tests/test_gpu_binned.py tests/test_gpu_margin.py -x -q > gpurun_out/r2i/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2i/pytest.log
timeout 1800 python tools/exp_c3res.py c3 1e9 0 6.5 > gpurun_out/r2i/c3res.log 2>&1; echo rc=$? >> gpurun_out/r2i/c3res.log
