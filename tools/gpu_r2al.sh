# r2al: pipelined scatter (cp.async double buffer, 1 CTA/SM) + coalesced unbin (pos16 + run table): binned tests, A/B vs old, launch list
mkdir -p gpurun_out/r2al
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2al/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2al/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2al/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1200 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_old.so $V/lib_op8.so $V/lib_ot512p16.so $V/lib_oub4.so $V/lib_s512x8.so $V/lib_s512x4.so $V/lib_u256.so $V/lib_u1024.so $V/lib_old.so > gpurun_out/r2al/ab_c3.log 2>&1
timeout 600 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_old.so $V/lib_s512x8.so $V/lib_old.so > gpurun_out/r2al/ab_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced" --csv --log-file gpurun_out/r2al/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2al/ncu.log 2>&1
