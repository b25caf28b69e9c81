# r2aw: double slots staged through the pools (16 per batch) instead of 16 direct 16-byte loads per lane: binned + parity tests, A/B c3/c4, launch list
mkdir -p gpurun_out/r2aw
timeout 900 python -m pytest tests/test_gpu_binned.py tests/test_gpu_parity.py -x -q > gpurun_out/r2aw/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2aw/pytest.log
V=paper_2005_03156_b200/_lib/var
timeout 1500 python tools/exp_variants.py c3 1e9 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2aw/ab_c3.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 $V/lib_prev.so $V/lib_prev.so > gpurun_out/r2aw/ab_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,l1tex__t_requests.sum,l1tex__data_pipe_lsu_wavefronts.sum --clock-control none \
  -k regex:"binned_query" --csv --log-file gpurun_out/r2aw/launches.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2aw/ncu.log 2>&1
