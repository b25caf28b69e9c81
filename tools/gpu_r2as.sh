# r2as: shared-memory scatter + run-table gather + half-slot ring: full GPU suite, smoke, bench, c3 launch list
mkdir -p gpurun_out/r2as
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2as/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2as/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2as/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2as/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2as/smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/r2as/bench.log 2>&1; echo rc=$? >> gpurun_out/r2as/bench.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --check-points 1000000"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|stream_kernel|resolve_kernel|widen" --csv --log-file gpurun_out/r2as/launches_c3.csv $CMD > gpurun_out/r2as/ncu_l.log 2>&1; echo rc=$? >> gpurun_out/r2as/ncu_l.log
