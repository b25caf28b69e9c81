# r2ar: binned query: L2 prefetch of slots at ring entry (doubles / all), points per lane per tile (1, 2, 3)
mkdir -p gpurun_out/r2ar
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_pf1.so $V/lib_pf2.so $V/lib_ku1.so $V/lib_ku3.so $V/lib_pf1.so $V/lib_pf2.so $V/lib_ku1.so $V/lib_ku3.so > gpurun_out/r2ar/ab_c3.log 2>&1
