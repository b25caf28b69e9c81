# r2bp: unbin CTA shapes at 32 registers (4 x 512 default, 8 x 256, 2 x 1024)
mkdir -p gpurun_out/r2bp
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_prev.so $V/lib_u256m8.so $V/lib_u1024m2.so $V/lib_prev.so > gpurun_out/r2bp/ab_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2bp/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bp/pytest.log
