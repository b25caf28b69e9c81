# r2bz: c3 grid resolution x tile size with the final kernels (cells per leaf side 6, 7, 8; tiles of 64 MB and 256 MB)
mkdir -p gpurun_out/r2bz
EXP_TILES="64e6 256e6" timeout 1800 python tools/exp_c3res.py c3 1e9 0 7 8 > gpurun_out/r2bz/c3res.log 2>&1
