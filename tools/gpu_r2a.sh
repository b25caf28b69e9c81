# round-2 baseline: c3 at 1B points (the N=1 headline config), c4 at 200M, launch list of c3
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2a/gpu.txt 2>&1
nproc >> gpurun_out/r2a/gpu.txt; free -g >> gpurun_out/r2a/gpu.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/r2a/gpu.txt
( time timeout 1500 python bench.py --config c3 --points 1000000000 --no-cpu --no-e2e --steps 5 ) > gpurun_out/r2a/c3_1B.log 2>&1; echo rc=$? >> gpurun_out/r2a/c3_1B.log
( time timeout 900 python bench.py --config c4 --no-cpu --no-e2e --steps 5 ) > gpurun_out/r2a/c4.log 2>&1; echo rc=$? >> gpurun_out/r2a/c4.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/r2a/launches_c3.csv \
  python bench.py --config c3 --points 1000000000 --no-cpu --no-e2e --steps 1 --warmup 0 > gpurun_out/r2a/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/r2a/ncu_c3.log
