# r2ay: edge_bit with one selected base point (fmin/fmax latitudes, D or -D): full GPU suite (bit-exactness), A/B c3/c4/c2
mkdir -p gpurun_out/r2ay
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2ay/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ay/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2ay/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2ay/ab_c4.log 2>&1
timeout 900 python tools/exp_variants.py c2 1e8 stream 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2ay/ab_c2.log 2>&1
