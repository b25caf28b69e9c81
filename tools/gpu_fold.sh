# folded query grid: GPU tests + c2/c4 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fold_pytest.log 2>&1; echo pytest=$? >> gpurun_out/fold_pytest.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/fold_bench_c2.log 2>&1; echo bench=$? >> gpurun_out/fold_bench_c2.log
timeout 600 python bench.py --no-cpu --no-e2e --config c4 --points 100000000 > gpurun_out/fold_bench_c4.log 2>&1; echo bench=$? >> gpurun_out/fold_bench_c4.log
timeout 600 python bench.py --no-cpu --no-e2e --mode approx --epsilon 5e-3 > gpurun_out/fold_bench_approx.log 2>&1; echo bench=$? >> gpurun_out/fold_bench_approx.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/launches_fold.csv $CMD > gpurun_out/ncu_l_fold.log 2>&1
