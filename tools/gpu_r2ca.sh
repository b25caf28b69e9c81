# r2ca: c3 at 7 / 8 cells per leaf side without the query-side fold (flat grid, as the binned path wants it)
mkdir -p gpurun_out/r2ca
FASTMAP_B200_LIB=$PWD/paper_2005_03156_b200/_lib/var/lib_nofold.so EXP_TILES="64e6" timeout 1800 python tools/exp_c3res.py c3 1e9 0 7 8 9 > gpurun_out/r2ca/c3res_nofold.log 2>&1
