SWEEP_MS="0" bash tools/gpu_ab.sh ab18
for v in default paper_2005_03156_b200/_lib/var/lib_b3.so paper_2005_03156_b200/_lib/var/lib_b4.so paper_2005_03156_b200/_lib/var/lib_w4b4.so; do
  if [ $v = default ]; then SWEEP_CONFIG=c4 timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/ab18_c4.log 2>&1;
  else FASTMAP_B200_LIB=$v SWEEP_CONFIG=c4 timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/ab18_c4.log 2>&1; fi
done
