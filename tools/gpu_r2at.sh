# r2at: binned query warps per CTA (2 CTAs/SM x 8..12 warps; 96 registers without spills at 10)
mkdir -p gpurun_out/r2at
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_qw9.so $V/lib_qw10.so $V/lib_qw11.so $V/lib_qw12.so $V/lib_qw9.so $V/lib_qw10.so $V/lib_qw11.so $V/lib_qw12.so > gpurun_out/r2at/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_qw10.so $V/lib_qw12.so $V/lib_qw10.so > gpurun_out/r2at/ab_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" --csv --log-file gpurun_out/r2at/launches_c4.csv python tools/exp_binned.py c4 2e8 0 > gpurun_out/r2at/ncu_c4.log 2>&1
