# r2bw: the stream path's slot staging with the binned path's cheap addresses: parity tests, A/B on c2, c1 and c3/c4 (stream path)
mkdir -p gpurun_out/r2bw
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_margin.py -x -q > gpurun_out/r2bw/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bw/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 900 python tools/exp_variants.py c2 1e8 stream 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bw/ab_c2.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 stream 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bw/ab_c4s.log 2>&1
timeout 900 python tools/exp_variants.py c1 1e8 stream 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bw/ab_c1.log 2>&1
