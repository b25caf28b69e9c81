# tuning variants of the product library (same sources, different -D knobs)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2005_03156_b200/_lib/var
for v in "$@"; do
  # v like W8_U2_P3072
  W=$(echo $v | sed 's/W\([0-9]*\)_.*/\1/'); U=$(echo $v | sed 's/.*_U\([0-9]*\)_.*/\1/'); P=$(echo $v | sed 's/.*_P\([0-9]*\)/\1/')
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -DFM_BWARPS=$W -DFM_KU=$U -DFM_BPOOL=$P -Xcompiler -fPIC,-O3,-ffp-contract=off,-pthread -shared \
    paper_2005_03156_b200/csrc/fastmap_b200.cu paper_2005_03156_b200/csrc/index_host.cpp \
    -o paper_2005_03156_b200/_lib/var/lib_$v.so &
done
wait
