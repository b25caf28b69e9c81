# all GPU tests, then the c2 sweep for the default library and every variant in _lib/var
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/var_pytest.log 2>&1; echo pytest=$? >> gpurun_out/var_pytest.log
timeout 300 python tools/exp_sweep.py 0 > gpurun_out/var_sweep.log 2>&1
for v in paper_2005_03156_b200/_lib/var/*.so; do
  FASTMAP_B200_LIB=$v timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/var_sweep.log 2>&1
done
