set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 600 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-e2e --points 20000000 > gpurun_out/bench_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:project_kernel --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-e2e --points 20000000 > gpurun_out/ncu1.log 2>&1; echo ncu=$?
