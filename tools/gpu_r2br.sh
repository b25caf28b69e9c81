# r2br: scatter at 2 x 1024 threads per SM (32 registers, 64 warps) against 2 x 512
mkdir -p gpurun_out/r2br
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_s1024m2.so $V/lib_s1024m2.so > gpurun_out/r2br/ab_c3.log 2>&1
FASTMAP_B200_LIB=$PWD/$V/lib_s1024m2.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_scatter" --csv --log-file gpurun_out/r2br/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2br/ncu.log 2>&1
