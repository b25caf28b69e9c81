# r2bh: how the binned kernels scale with resident CTAs per SM (query 1 vs 2, scatter 1 vs 2, unbin 1/2 vs 4): ncu launch lists
mkdir -p gpurun_out/r2bh
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum"
FM_DBG_QGRID=148 FM_DBG_SGRID=148 FM_DBG_UGRID=148 timeout 900 ncu --metrics $M --clock-control none -k regex:"bin_scatter|binned_query|unbin" --csv --log-file gpurun_out/r2bh/launches_1.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bh/ncu1.log 2>&1
FM_DBG_UGRID=296 FM_DBG_QGRID=222 timeout 900 ncu --metrics $M --clock-control none -k regex:"bin_scatter|binned_query|unbin" --csv --log-file gpurun_out/r2bh/launches_2.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bh/ncu2.log 2>&1
