timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t10_pytest.log 2>&1; echo pytest=$? >> gpurun_out/t10_pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/t10_bench.json 2> gpurun_out/t10_bench.err
SWEEP_CONFIG=c4 timeout 600 python tools/exp_sweep.py 0 >> gpurun_out/t10_c4.log 2>&1
SWEEP_CONFIG=c1 timeout 600 python tools/exp_sweep.py 0 >> gpurun_out/t10_c1.log 2>&1
