# one GPU iteration: parity tests, c2 bench, full ncu capture of the kernel
TAG=${1:-iter}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu ${BENCH_EXTRA} > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
if [ "${NCU:-1}" = "1" ]; then
timeout 600 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-e2e --points 20000000 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:project_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-e2e --points 20000000 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu=$?
fi
