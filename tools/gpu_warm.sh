# warm-cache per-kernel times (ncu --cache-control none) for the folded and flat query grids
mkdir -p gpurun_out
timeout 300 ./oracle/_ref/adapter_check gpu > gpurun_out/warm_adapter.log 2>&1; echo rc=$? >> gpurun_out/warm_adapter.log
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/warm_plain.log 2>&1
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/warm_fold.csv $CMD > gpurun_out/warm_fold.log 2>&1
FASTMAP_B200_LIB=paper_2005_03156_b200/_lib/var/lib_flat.so timeout 300 $CMD > gpurun_out/warm_plain_flat.log 2>&1
FASTMAP_B200_LIB=paper_2005_03156_b200/_lib/var/lib_flat.so timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/warm_flat.csv $CMD > gpurun_out/warm_flat.log 2>&1
