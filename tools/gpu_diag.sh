mkdir -p gpurun_out
SWEEP_CONFIG=c2 timeout 600 python tools/exp_sweep.py 8 9 10 11 12 14 > gpurun_out/diag_m.log 2>&1
