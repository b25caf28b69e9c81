# r2bq: scatter placement pass without the overflow branch when no run of the chunk overflowed (bounds test kept)
mkdir -p gpurun_out/r2bq
V=paper_2005_03156_b200/_lib/var
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_scatter" --csv --log-file gpurun_out/r2bq/launches_noovf.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bq/ncu1.log 2>&1
FASTMAP_B200_LIB=$PWD/$V/lib_gen.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_scatter" --csv --log-file gpurun_out/r2bq/launches_gen.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bq/ncu2.log 2>&1
