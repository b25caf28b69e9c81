# r2h: barrier-free scatter + unbin variants on c3 (1B points), per-kernel launch list
mkdir -p gpurun_out/r2h
V="paper_2005_03156_b200/_lib/var/lib_r4.so paper_2005_03156_b200/_lib/var/lib_cg8.so paper_2005_03156_b200/_lib/var/lib_r2.so"
timeout 900 python tools/exp_variants.py c3 1e9 binned 128e6 $V > gpurun_out/r2h/var_630.log 2>&1; echo rc=$? >> gpurun_out/r2h/var_630.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin" --csv --log-file gpurun_out/r2h/launches_c3.csv \
  python tools/exp_binned.py c3 1e9 32e6 128e6 > gpurun_out/r2h/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/r2h/ncu_c3.log
