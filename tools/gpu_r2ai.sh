# r2ai: sampled binning with per-thread bin claims: A/B vs the counting pass (c3 default and m=6), launch list
mkdir -p gpurun_out/r2ai
V=paper_2005_03156_b200/_lib/var
timeout 900 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_count.so $V/lib_sample.so $V/lib_count.so $V/lib_sample.so > gpurun_out/r2ai/ab_c3.log 2>&1
EXPV_M=6 timeout 900 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_count.so $V/lib_sample.so $V/lib_count.so $V/lib_sample.so > gpurun_out/r2ai/ab_c3m6.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" -c 14 --csv --log-file gpurun_out/r2ai/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2ai/ncu.log 2>&1
