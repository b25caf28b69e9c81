# r2ag: full ncu captures (source-level) of the binned query kernel at the default c3 resolution and at m=6
mkdir -p gpurun_out/r2ag
for M in 0 6; do
EXP_TILES="0" timeout 900 ncu --set full --import-source on --clock-control none -k regex:binned_query --launch-skip 1 -c 1 \
  -o gpurun_out/r2ag/q_m$M python tools/exp_c3res.py c3 1e9 $M > gpurun_out/r2ag/ncu_m$M.log 2>&1
done
