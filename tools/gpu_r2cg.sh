# r2cg: points per lane per tile (1, 2, 3) at the final defaults
mkdir -p gpurun_out/r2cg
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_ku3.so $V/lib_ku1.so $V/lib_ku3.so > gpurun_out/r2cg/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_ku3.so $V/lib_ku1.so > gpurun_out/r2cg/ab_c4.log 2>&1
