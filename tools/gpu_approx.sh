# fast-approx mode on the GPU: tests, C++ adapter (incl. approx), bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_approx.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/approx_pytest.log 2>&1; echo pytest=$? >> gpurun_out/approx_pytest.log
timeout 300 ./oracle/_ref/adapter_check gpu > gpurun_out/approx_adapter.log 2>&1; echo adapter=$? >> gpurun_out/approx_adapter.log
timeout 600 python bench.py --mode approx --epsilon 5e-3 --no-cpu --no-e2e > gpurun_out/approx_bench_c2.log 2>&1; echo bench=$? >> gpurun_out/approx_bench_c2.log
timeout 600 python bench.py --mode approx --epsilon 2e-3 --no-cpu --no-e2e > gpurun_out/approx_bench_c2_2e3.log 2>&1; echo bench=$? >> gpurun_out/approx_bench_c2_2e3.log
timeout 600 python bench.py --mode approx --epsilon 2e-2 --no-cpu --no-e2e > gpurun_out/approx_bench_c2_2e2.log 2>&1; echo bench=$? >> gpurun_out/approx_bench_c2_2e2.log
