# r2ax: full ncu capture (source-level) of the binned query kernel with half / staged double rings on c3
mkdir -p gpurun_out/r2ax
EXP_TILES="0" timeout 900 ncu --set full --import-source on --clock-control none -k regex:binned_query --launch-skip 1 -c 1 \
  -o gpurun_out/r2ax/bq python tools/exp_c3res.py c3 1e9 0 > gpurun_out/r2ax/ncu.log 2>&1
