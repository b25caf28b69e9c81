SWEEP_MS="0" bash tools/gpu_ab.sh ab16
for r in 1 1:0.5 1:0.3; do FASTMAP_B200_L2PERSIST=$r SWEEP_LIB_TAG=l2p$r timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/ab16_sweep.log 2>&1; done
