# r2bc: tile groups per work-counter grab in the binned query (4, 8, 16, 32)
mkdir -p gpurun_out/r2bc
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_g4.so $V/lib_g16.so $V/lib_g32.so $V/lib_g4.so $V/lib_g16.so $V/lib_g32.so > gpurun_out/r2bc/ab_c3.log 2>&1
