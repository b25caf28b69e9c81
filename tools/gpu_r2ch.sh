# r2ch: where the binned path starts to pay: stream vs binned at 2M..32M points on c4 and c3
mkdir -p gpurun_out/r2ch
for N in 2e6 4e6 8e6 16e6 32e6; do
timeout 600 python tools/exp_binned.py c4 $N 0 >> gpurun_out/r2ch/c4.log 2>&1
done
for N in 4e6 8e6 16e6 32e6; do
timeout 600 python tools/exp_binned.py c3 $N 0 >> gpurun_out/r2ch/c3.log 2>&1
done
