# A/B: current library vs _lib/var/lib_prev.so on c2 and c4, alternating, then again after a pytest pass
mkdir -p gpurun_out
ab() {
  for r in 1 2; do
    timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/ab_$1_cur_$r.log 2>&1
    FASTMAP_B200_LIB=paper_2005_03156_b200/_lib/var/lib_prev.so timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/ab_$1_prev_$r.log 2>&1
  done
  timeout 600 python bench.py --no-cpu --no-e2e --config c4 --points 100000000 > gpurun_out/ab_$1_cur_c4.log 2>&1
  FASTMAP_B200_LIB=paper_2005_03156_b200/_lib/var/lib_prev.so timeout 600 python bench.py --no-cpu --no-e2e --config c4 --points 100000000 > gpurun_out/ab_$1_prev_c4.log 2>&1
}
ab a
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_build.py -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1
ab b
