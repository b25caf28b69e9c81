# r2bg: sampling stride of the bin-capacity estimate (64, 128, 256, 512)
mkdir -p gpurun_out/r2bg
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_s128.so $V/lib_s256.so $V/lib_s512.so $V/lib_s128.so $V/lib_s256.so $V/lib_s512.so > gpurun_out/r2bg/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_s128.so $V/lib_s256.so $V/lib_s512.so > gpurun_out/r2bg/ab_c4.log 2>&1
