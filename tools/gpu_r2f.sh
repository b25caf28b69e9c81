# r2f: full ncu captures of the binned path's kernels on c3 (1B points), and the
# c3 launch list of the default bench command (roofline.traffic for c3)
mkdir -p gpurun_out/r2f
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bin_scatter|binned_query|unbin|bin_count" -c 4 \
  -o gpurun_out/r2f/prof_binned python tools/exp_binned.py c3 1e9 32e6 > gpurun_out/r2f/ncu_full.log 2>&1; echo rc=$? >> gpurun_out/r2f/ncu_full.log
for k in bin_count_kernel bin_scatter_kernel binned_query_kernel unbin_kernel; do
  ncu -i gpurun_out/r2f/prof_binned.ncu-rep --page raw --csv -k regex:$k > gpurun_out/r2f/raw_$k.csv 2>/dev/null
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --check-points 1000000"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel|bin_|binned|unbin" --csv --log-file gpurun_out/r2f/launches_c3.csv $CMD > gpurun_out/r2f/ncu_l.log 2>&1; echo rc=$? >> gpurun_out/r2f/ncu_l.log
