# quick GPU check: parity tests + sweep (each step under its own timeout)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo pytest=$? >> gpurun_out/pytest_quick.log
timeout 300 python tools/exp_sweep.py 0 > gpurun_out/sweep_quick.log 2>&1; echo sweep=$? >> gpurun_out/sweep_quick.log
for v in $(ls paper_2005_03156_b200/_lib/var/*.so 2>/dev/null); do
  FASTMAP_B200_LIB=$v timeout 300 python tools/exp_sweep.py 0 >> gpurun_out/sweep_quick_var.log 2>&1
done
