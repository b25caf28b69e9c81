# r2ce: final state of round 2 (flat grid on the binned path, c3 at 8 cells per leaf side, cap 64): full GPU suite, smoke, bench (c3), reference arm, c3 launch list, other configs
mkdir -p gpurun_out/r2ce
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2ce/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2ce/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ce/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ce/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2ce/smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/r2ce/bench.log 2>&1; echo rc=$? >> gpurun_out/r2ce/bench.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --check-points 1000000"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced|stream_kernel|resolve_kernel" --csv --log-file gpurun_out/r2ce/launches_c3.csv $CMD > gpurun_out/r2ce/ncu_l.log 2>&1; echo rc=$? >> gpurun_out/r2ce/ncu_l.log
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/r2ce/benchref.log 2>&1; echo rc=$? >> gpurun_out/r2ce/benchref.log
timeout 600 python bench.py --config c2 --no-cpu --no-e2e > gpurun_out/r2ce/c2.log 2>&1
timeout 600 python bench.py --config c2 --hist --no-cpu --no-e2e > gpurun_out/r2ce/c2_hist.log 2>&1
timeout 600 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/r2ce/c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --no-cpu --no-e2e --check-points 2000000 > gpurun_out/r2ce/c5.log 2>&1
