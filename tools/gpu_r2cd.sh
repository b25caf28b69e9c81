# r2cd: c4 grid resolution with the flat query grid (48 default, 64, 80, 96 cells per polygon side)
mkdir -p gpurun_out/r2cd
EXP_TILES="64e6" timeout 1500 python tools/exp_c3res.py c4 2e8 0 64 80 96 > gpurun_out/r2cd/c4res.log 2>&1
