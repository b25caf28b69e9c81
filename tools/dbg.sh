for v in default paper_2005_03156_b200/_lib/var/lib_xu2.so paper_2005_03156_b200/_lib/var/lib_xu8.so paper_2005_03156_b200/_lib/var/lib_head2.so; do
  for pass in 1 2; do
  if [ $v = default ]; then timeout 600 python bench.py --mode approx --no-cpu --no-e2e > gpurun_out/ax_$(basename $v)_$pass.log 2>&1;
  else FASTMAP_B200_LIB=$v timeout 600 python bench.py --mode approx --no-cpu --no-e2e > gpurun_out/ax_$(basename $v)_$pass.log 2>&1; fi
  done
done
timeout 300 python -m pytest tests/test_gpu_approx.py -m gpu -x -q > gpurun_out/ax_pytest.log 2>&1; echo rc=$? >> gpurun_out/ax_pytest.log
