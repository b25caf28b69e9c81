# r2aa: binned histogram variants (aggregation, chunk sizes); reference max_level sweep (c2, c3)
mkdir -p gpurun_out/r2aa
V="paper_2005_03156_b200/_lib/var/lib_agg.so paper_2005_03156_b200/_lib/var/lib_ch64.so paper_2005_03156_b200/_lib/var/lib_ch4.so"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"binned_hist" --csv --log-file gpurun_out/r2aa/launches_hist.csv \
  env EXPV_HIST=1 python tools/exp_variants.py c3 1e9 binned 0 $V > gpurun_out/r2aa/ncu.log 2>&1
timeout 1500 python tools/ref_sweep.py c2 20e6 12 14 16 18 > gpurun_out/r2aa/ref_c2.log 2>&1
timeout 1500 python tools/ref_sweep.py c3 20e6 12 14 16 > gpurun_out/r2aa/ref_c3.log 2>&1
