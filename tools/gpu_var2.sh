# bench vs sweep at the default resolution, repeated, same box
mkdir -p gpurun_out
for r in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/v2_bench_$r.log 2>&1
timeout 600 python tools/exp_sweep.py 0 25 > gpurun_out/v2_sweep_$r.log 2>&1
done
