# r2bb: grid-resolution sweeps with the round's final kernels: c3 (cells per leaf side 5..8), c4 (cells per polygon side 36..80), binned path only
mkdir -p gpurun_out/r2bb
EXP_TILES="0" EXP_NO_STREAM=1 timeout 1500 python tools/exp_c3res.py c3 1e9 0 5 7 8 > gpurun_out/r2bb/c3res.log 2>&1
EXP_TILES="0" EXP_NO_STREAM=1 timeout 1200 python tools/exp_c3res.py c4 2e8 0 36 56 64 80 > gpurun_out/r2bb/c4res.log 2>&1
