# FP64 microbenchmark (tools/exp_fp64.cu), compiled and run on the box
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false tools/exp_fp64.cu -o gpurun_out/exp_fp64 && \
for r in 1 2 3; do timeout 120 ./gpurun_out/exp_fp64; done > gpurun_out/fp64.jsonl 2>&1
rm -f gpurun_out/exp_fp64
