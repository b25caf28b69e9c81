# Full GPU round: tests, smoke, bench (ours + reference arm), ncu launch list
# and full captures of both kernels.  Every step under its own timeout.
TAG=${1:-round}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
nproc >> gpurun_out/gpu_$TAG.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/benchref_$TAG.json 2> gpurun_out/benchref_$TAG.err; echo "ref rc=$?" >> gpurun_out/benchref_$TAG.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_l_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|resolve_kernel" -s 6 -c 2 \
  -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
# fast-approx leg: bench line + launch list of approx_kernel
ACMD="python bench.py --mode approx --epsilon 5e-3 --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 600 python bench.py --mode approx --epsilon 5e-3 --no-cpu > gpurun_out/bench_approx_$TAG.json 2> gpurun_out/bench_approx_$TAG.err
timeout 300 $ACMD > gpurun_out/plain_approx_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"approx_kernel" --csv --log-file gpurun_out/launches_approx_$TAG.csv $ACMD > gpurun_out/ncu_la_$TAG.log 2>&1
echo "approx ncu rc=$?" >> gpurun_out/ncu_la_$TAG.log
