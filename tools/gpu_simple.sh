# simple engine + IO GPU tests, then simple-engine bench lines (c3s)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_simple.py tests/test_gpu_io.py -m gpu -x -q > gpurun_out/simple_pytest.log 2>&1; echo pytest=$? >> gpurun_out/simple_pytest.log
timeout 900 python bench.py --config c3s --mode simple --no-cpu > gpurun_out/simple_bench.log 2>&1; echo rc=$? >> gpurun_out/simple_bench.log
timeout 900 python bench.py --config c3s --mode simple-strict --no-cpu --no-e2e > gpurun_out/simple_strict_bench.log 2>&1; echo rc=$? >> gpurun_out/simple_strict_bench.log
timeout 900 python bench.py --config c3s --no-cpu --no-e2e > gpurun_out/c3s_exact_bench.log 2>&1; echo rc=$? >> gpurun_out/c3s_exact_bench.log
