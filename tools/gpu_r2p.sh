# r2p: scatter cost decomposition (variant libraries, ncu per-launch durations of bin_scatter)
mkdir -p gpurun_out/r2p
V="paper_2005_03156_b200/_lib/var/lib_noatom.so paper_2005_03156_b200/_lib/var/lib_nostore.so paper_2005_03156_b200/_lib/var/lib_noboth.so paper_2005_03156_b200/_lib/var/lib_per8.so"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none \
  -k regex:"bin_scatter" --csv --log-file gpurun_out/r2p/launches.csv \
  python tools/exp_variants.py c3 1e9 binned 64e6 $V > gpurun_out/r2p/var.log 2>&1; echo rc=$? >> gpurun_out/r2p/var.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bin_scatter" -c 1 \
  -o gpurun_out/r2p/prof python tools/exp_binned.py c3 2e8 64e6 > gpurun_out/r2p/ncu_full.log 2>&1; echo rc=$? >> gpurun_out/r2p/ncu_full.log
