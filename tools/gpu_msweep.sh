# resolution sweeps per config (default library), for the default cell budget
TAG=${1:-ms}
mkdir -p gpurun_out
SWEEP_POINTS=100000000 timeout 600 python tools/exp_sweep.py 0 40 48 56 64 >> gpurun_out/${TAG}_c2.log 2>&1
SWEEP_CONFIG=c4 timeout 600 python tools/exp_sweep.py 24 32 40 48 >> gpurun_out/${TAG}_c4.log 2>&1
SWEEP_CONFIG=c1 timeout 600 python tools/exp_sweep.py 32 40 64 >> gpurun_out/${TAG}_c1.log 2>&1
