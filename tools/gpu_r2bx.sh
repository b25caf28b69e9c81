# r2bx: final state of round 2: full GPU suite, smoke, bench (c3), reference arm, c3 launch list, other configs, a two-batch call (2^30 + 1000 points)
mkdir -p gpurun_out/r2bx
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2bx/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bx/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2bx/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bx/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2bx/smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/r2bx/bench.log 2>&1; echo rc=$? >> gpurun_out/r2bx/bench.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --check-points 1000000"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"bin_|binned|unbin|unplaced|stream_kernel|resolve_kernel" --csv --log-file gpurun_out/r2bx/launches_c3.csv $CMD > gpurun_out/r2bx/ncu_l.log 2>&1; echo rc=$? >> gpurun_out/r2bx/ncu_l.log
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/r2bx/benchref.log 2>&1; echo rc=$? >> gpurun_out/r2bx/benchref.log
timeout 600 python bench.py --config c2 --no-cpu --no-e2e > gpurun_out/r2bx/c2.log 2>&1
timeout 600 python bench.py --config c2 --hist --no-cpu --no-e2e > gpurun_out/r2bx/c2_hist.log 2>&1
timeout 600 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/r2bx/c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --no-cpu --no-e2e --check-points 2000000 > gpurun_out/r2bx/c5.log 2>&1
timeout 900 python tools/exp_binned.py c3 1073742824 0 > gpurun_out/r2bx/two_batches.log 2>&1
