# r2cc: tile size at the new c3 default (8 cells per leaf side, flat grid): 64 MB (480 tiles) vs 256 MB (120 tiles); c3 at 8.5 cells per side
mkdir -p gpurun_out/r2cc
timeout 900 python tools/exp_binned.py c3 1e9 64e6 256e6 > gpurun_out/r2cc/tiles.log 2>&1
EXP_TILES="64e6" timeout 1200 python tools/exp_c3res.py c3 1e9 8.5 > gpurun_out/r2cc/c3res.log 2>&1
timeout 900 python tools/exp_binned.py c4 2e8 64e6 16e6 256e6 > gpurun_out/r2cc/tiles_c4.log 2>&1
