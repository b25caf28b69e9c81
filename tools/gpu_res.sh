# resolution sweep (two interleaved passes) for c2 and c4
mkdir -p gpurun_out
timeout 1200 python tools/exp_sweep.py 22 25 28 32 22 25 28 32 > gpurun_out/res2_sweep.log 2>&1
SWEEP_CONFIG=c4 timeout 1200 python tools/exp_sweep.py 28 32 40 45 28 32 40 45 >> gpurun_out/res2_sweep.log 2>&1
