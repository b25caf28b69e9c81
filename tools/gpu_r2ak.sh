# r2ak: slot staging A/B (old per-copy address arithmetic vs precomputed swizzle/predicates), c3 and c4
mkdir -p gpurun_out/r2ak
V=paper_2005_03156_b200/_lib/var
timeout 900 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_old.so $V/lib_new.so $V/lib_old.so $V/lib_new.so > gpurun_out/r2ak/ab_c3.log 2>&1
timeout 600 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_old.so $V/lib_new.so $V/lib_old.so $V/lib_new.so > gpurun_out/r2ak/ab_c4.log 2>&1
timeout 600 python tools/exp_variants.py c2 1e8 stream 0 $V/lib_old.so $V/lib_new.so $V/lib_old.so $V/lib_new.so > gpurun_out/r2ak/ab_c2.log 2>&1
