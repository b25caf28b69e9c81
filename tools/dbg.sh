SWEEP_MS="0" bash tools/gpu_ab.sh ab14
SWEEP_CONFIG=c1 timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/ab14_sweep.log 2>&1
FASTMAP_B200_LIB=paper_2005_03156_b200/_lib/var/lib_prev.so SWEEP_CONFIG=c1 timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/ab14_sweep.log 2>&1
