# all GPU tests + bench lines (c2 exact / approx, c4, c1) + c2 launch list; TAG names the logs
TAG=${1:-chk}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c2.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --config c4 --points 100000000 > gpurun_out/${TAG}_bench_c4.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --config c1 --points 100000000 > gpurun_out/${TAG}_bench_c1.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --mode approx --epsilon 5e-3 > gpurun_out/${TAG}_bench_approx.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_l_${TAG}.log 2>&1
