# r2am: unbin2 with run-head flags + warp scan (no per-point search), scatter2 buffer/CTA shapes, binned query at 3-4 CTAs/SM (one slot pool per warp)
mkdir -p gpurun_out/r2am
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2am/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2am/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_old.so $V/lib_sb1.so $V/lib_s512x8.so $V/lib_qD.so $V/lib_qA.so $V/lib_qB.so $V/lib_qC.so $V/lib_u256.so $V/lib_u1024.so $V/lib_old.so > gpurun_out/r2am/ab_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" --csv --log-file gpurun_out/r2am/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2am/ncu.log 2>&1
