# tuning variants of the product library: args like B8_U2_M3 (resolve warps,
# stream points per lane, resolve min blocks per SM for __launch_bounds__)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2005_03156_b200/_lib/var
for v in "$@"; do
  B=$(echo $v | sed 's/B\([0-9]*\)_.*/\1/'); U=$(echo $v | sed 's/.*_U\([0-9]*\)_.*/\1/'); M=$(echo $v | sed 's/.*_M\([0-9]*\)/\1/')
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -DFM_BWARPS=$B -DFM_KU=$U -DFM_BMINB=$M -Xcompiler -fPIC,-O3,-ffp-contract=off,-pthread -shared \
    paper_2005_03156_b200/csrc/fastmap_b200.cu paper_2005_03156_b200/csrc/index_gpu.cu paper_2005_03156_b200/csrc/index_host.cpp \
    -o paper_2005_03156_b200/_lib/var/lib_$v.so -Xptxas -v 2> paper_2005_03156_b200/_lib/var/ptxas_$v.log &
done
wait
