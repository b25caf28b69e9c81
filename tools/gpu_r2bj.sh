# r2bj: binned query at 3 CTAs x 6 warps with __maxnreg__ 112 / 104 (103 / 99 registers, no spills)
mkdir -p gpurun_out/r2bj
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_w6r112.so $V/lib_w6r104.so $V/lib_w8r120.so > gpurun_out/r2bj/ab_c3.log 2>&1
