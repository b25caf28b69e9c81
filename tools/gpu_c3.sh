# c3 / c5 at scale on one GPU: the 12.5M-leaf c3 index built on the GPU, then
# bench lines for c3 (200M points per step) and c5 (1B points per GPU per
# step with the int64 per-block histogram), each under its own timeout
mkdir -p gpurun_out
timeout 2400 python bench.py --config c3 --points 200000000 --no-cpu --no-e2e --steps 5 > gpurun_out/c3_bench.log 2>&1; echo rc=$? >> gpurun_out/c3_bench.log
timeout 3000 python bench.py --config c5 --points 1000000000 --hist --no-cpu --no-e2e --steps 3 > gpurun_out/c5_bench.log 2>&1; echo rc=$? >> gpurun_out/c5_bench.log
