# r2ae: c3 grid resolution with the round-2 pipeline (double slots, binned path)
mkdir -p gpurun_out/r2ae
EXP_TILES="0" timeout 2400 python tools/exp_c3res.py c3 1e9 0 5.5 6.5 8 > gpurun_out/r2ae/c3res.log 2>&1
