# r2aq: point-load cache policy of the binned query with the half ring (ld.cs vs ld.nc vs ld.ca): c3 A/B, launch list with ldg
mkdir -p gpurun_out/r2aq
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_qh0.so $V/lib_ldg.so $V/lib_ldca.so $V/lib_qh0.so $V/lib_ldg.so $V/lib_ldca.so > gpurun_out/r2aq/ab_c3.log 2>&1
FASTMAP_B200_LIB=$PWD/$V/lib_ldg.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"binned" --csv --log-file gpurun_out/r2aq/launches_ldg.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2aq/ncu.log 2>&1
