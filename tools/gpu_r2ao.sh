# r2ao: scatter2 CTA shapes (3 x 384 threads / chunk 3072, 4 x 256 / chunk 2048, 2 x 256 x 16), tile-size sweep with the new scatter
mkdir -p gpurun_out/r2ao
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_s384m3.so $V/lib_s256m4.so $V/lib_s256p16.so $V/lib_u256.so > gpurun_out/r2ao/ab_c3.log 2>&1
timeout 1500 python tools/exp_binned.py c3 1e9 16e6 32e6 64e6 128e6 > gpurun_out/r2ao/tiles_c3.log 2>&1
