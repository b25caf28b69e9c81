timeout 300 python tools/dbg_quick.py c2 4000000 > gpurun_out/dbg19.log 2>&1
FASTMAP_B200_LIB=paper_2005_03156_b200/_lib/var/lib_a4.so timeout 300 python tools/dbg_quick.py c1 >> gpurun_out/dbg19.log 2>&1
SWEEP_MS="0" bash tools/gpu_ab.sh ab19
