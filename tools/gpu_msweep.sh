mkdir -p gpurun_out
timeout 600 python tools/exp_sweep.py 0 10 14 20 > gpurun_out/msweep.log 2>&1
SWEEP_CONFIG=c4 SWEEP_POINTS=50000000 timeout 600 python tools/exp_sweep.py 0 16 24 >> gpurun_out/msweep.log 2>&1
