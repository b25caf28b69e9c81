# r2af: c3 resolution x tile-size sweep (binned path), and per-kernel times at three resolutions
mkdir -p gpurun_out/r2af
EXP_TILES="0 24e6 40e6 96e6" timeout 2400 python tools/exp_c3res.py c3 1e9 5.0 5.5 6.0 7.0 > gpurun_out/r2af/c3res.log 2>&1
EXP_TILES="0" timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"bin_|binned|unbin" --csv --log-file gpurun_out/r2af/launches.csv python tools/exp_c3res.py c3 1e9 0 5.5 8 > gpurun_out/r2af/ncu.log 2>&1
