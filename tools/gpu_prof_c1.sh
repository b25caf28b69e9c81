mkdir -p gpurun_out
CMD="python bench.py --config c1 --points 100000000 --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain_c1.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_c1all.csv $CMD > gpurun_out/ncu_c1.log 2>&1
echo rc=$? >> gpurun_out/ncu_c1.log
