# r2bv: two lanes per double-slot item (edges 0-3 + candidates 0-3 / edges 4-8 + candidates 4-7): binned, parity, margin, build tests; A/B c3/c4
mkdir -p gpurun_out/r2bv
timeout 1200 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py tests/test_gpu_margin.py -x -q > gpurun_out/r2bv/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bv/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bv/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2bv/ab_c4.log 2>&1
