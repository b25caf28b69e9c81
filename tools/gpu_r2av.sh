# r2av: slot copies with cp.async.ca (L1-allocating) vs .cg: c3, c4, c2 (stream path)
mkdir -p gpurun_out/r2av
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_ca.so $V/lib_ca.so > gpurun_out/r2av/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_ca.so $V/lib_ca.so > gpurun_out/r2av/ab_c4.log 2>&1
timeout 900 python tools/exp_variants.py c2 1e8 stream 0 $V/lib_ca.so $V/lib_ca.so > gpurun_out/r2av/ab_c2.log 2>&1
FASTMAP_B200_LIB=$PWD/$V/lib_ca.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"binned_query" --csv --log-file gpurun_out/r2av/launches_ca.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2av/ncu.log 2>&1
