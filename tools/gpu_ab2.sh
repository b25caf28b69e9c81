# per-kernel warm times (ncu --cache-control none): current vs lib_prev
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/ab2_cur.csv $CMD > gpurun_out/ab2_cur.log 2>&1
FASTMAP_B200_LIB=paper_2005_03156_b200/_lib/var/lib_prev.so timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/ab2_prev.csv $CMD > gpurun_out/ab2_prev.log 2>&1
