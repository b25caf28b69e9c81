# r2bi: binned query CTA shapes at 3-5 CTAs per SM (6x3, 5x4, 4x5, 4x4 warps x CTAs)
mkdir -p gpurun_out/r2bi
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_w6b3.so $V/lib_w5b4.so $V/lib_w4b5.so $V/lib_w4b4.so > gpurun_out/r2bi/ab_c3.log 2>&1
