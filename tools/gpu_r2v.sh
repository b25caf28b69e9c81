# r2v: bench (c3 default, binned by auto), ncu launch list + full captures of the binned kernels,
# histogram overheads (c2, c5)
mkdir -p gpurun_out/r2v
( time timeout 1500 python bench.py ) > gpurun_out/r2v/bench.log 2>&1; echo rc=$? >> gpurun_out/r2v/bench.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --check-points 1000000"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|stream_kernel|resolve_kernel|widen" --csv --log-file gpurun_out/r2v/launches_c3.csv $CMD > gpurun_out/r2v/ncu_l.log 2>&1; echo rc=$? >> gpurun_out/r2v/ncu_l.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bin_scatter|binned_query|unbin|bin_count" -c 4 \
  -o gpurun_out/r2v/prof $CMD > gpurun_out/r2v/ncu_full.log 2>&1; echo rc=$? >> gpurun_out/r2v/ncu_full.log
timeout 600 python bench.py --config c2 --no-cpu --no-e2e > gpurun_out/r2v/c2.log 2>&1
timeout 600 python bench.py --config c2 --hist --no-cpu --no-e2e > gpurun_out/r2v/c2_hist.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --no-cpu --no-e2e --check-points 2000000 > gpurun_out/r2v/c5.log 2>&1
timeout 900 python bench.py --config c5 --hist --steps 3 --no-cpu --no-e2e --check-points 2000000 > gpurun_out/r2v/c5_hist.log 2>&1
