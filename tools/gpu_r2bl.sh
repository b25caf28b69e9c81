# r2bl: which of the scatter changes raised its L2 traffic (fp32 tile key vs the plain fast path)
mkdir -p gpurun_out/r2bl
V=paper_2005_03156_b200/_lib/var
for L in f64key noplain neither prev; do
FASTMAP_B200_LIB=$PWD/$V/lib_$L.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_scatter" --csv --log-file gpurun_out/r2bl/launches_$L.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bl/ncu_$L.log 2>&1
done
