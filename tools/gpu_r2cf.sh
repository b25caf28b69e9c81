# r2cf: full ncu capture (source-level) of the binned query kernel at the final defaults (c3, 8 cells per leaf side, flat grid)
mkdir -p gpurun_out/r2cf
EXP_TILES="0" timeout 900 ncu --set full --import-source on --clock-control none -k regex:binned_query --launch-skip 1 -c 1 \
  -o gpurun_out/r2cf/bq python tools/exp_c3res.py c3 1e9 0 > gpurun_out/r2cf/ncu.log 2>&1
