# r2an: full ncu capture (source-level) of bin_scatter2_kernel (2 CTAs x 512 threads, one window each) and unbin2_kernel on c3
mkdir -p gpurun_out/r2an
for K in bin_scatter2 unbin2; do
EXP_TILES="0" timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip 1 -c 1 \
  -o gpurun_out/r2an/$K python tools/exp_c3res.py c3 1e9 0 > gpurun_out/r2an/ncu_$K.log 2>&1
done
