# c2 + c4 sweeps (default resolution) for the default library and every _lib/var variant, two passes
mkdir -p gpurun_out
for pass in 1 2; do
  timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/variants_c2.log 2>&1
  for v in paper_2005_03156_b200/_lib/var/*.so; do
    FASTMAP_B200_LIB=$v timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/variants_c2.log 2>&1
  done
done
SWEEP_CONFIG=c4 timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/variants_c4.log 2>&1
for v in paper_2005_03156_b200/_lib/var/*.so; do
  SWEEP_CONFIG=c4 FASTMAP_B200_LIB=$v timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/variants_c4.log 2>&1
done
