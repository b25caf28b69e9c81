# half-slot layout: all GPU tests + exact bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/half_pytest.log 2>&1; echo pytest=$? >> gpurun_out/half_pytest.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/half_bench_c2.log 2>&1; echo bench=$? >> gpurun_out/half_bench_c2.log
timeout 600 python bench.py --no-cpu --no-e2e --config c4 --points 100000000 > gpurun_out/half_bench_c4.log 2>&1; echo bench=$? >> gpurun_out/half_bench_c4.log
timeout 300 python tools/exp_sweep.py 0 > gpurun_out/half_sweep.log 2>&1; echo sweep=$? >> gpurun_out/half_sweep.log
