# r2e: HEAD baseline at session start -- GPU tests, smoke, default bench (c3), reference arm
mkdir -p gpurun_out/r2e
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2e/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2e/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2e/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2e/smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/r2e/bench.log 2>&1; echo rc=$? >> gpurun_out/r2e/bench.log
( time timeout 1200 python bench.py --impl reference ) > gpurun_out/r2e/benchref.log 2>&1; echo rc=$? >> gpurun_out/r2e/benchref.log
