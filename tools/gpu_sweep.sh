mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_sweep.log 2>&1; echo pytest=$? >> gpurun_out/pytest_sweep.log
python tools/exp_sweep.py 0 > gpurun_out/sweep_default.log 2>&1
for v in paper_2005_03156_b200/_lib/var/*.so; do
  FASTMAP_B200_LIB=$v python tools/exp_sweep.py 0 >> gpurun_out/sweep_variants.log 2>&1
done
