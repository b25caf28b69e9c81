# r2bm: scatter with the no-overflow placement fast path and the looped write-out, against no fast path
mkdir -p gpurun_out/r2bm
V=paper_2005_03156_b200/_lib/var
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_scatter" --csv --log-file gpurun_out/r2bm/launches_plain.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bm/ncu_plain.log 2>&1
FASTMAP_B200_LIB=$PWD/$V/lib_noplain.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
  -k regex:"bin_scatter" --csv --log-file gpurun_out/r2bm/launches_noplain.csv python tools/exp_binned.py c3 1e9 0 > gpurun_out/r2bm/ncu_noplain.log 2>&1
timeout 900 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2bm/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bm/pytest.log
