# tuning variants of the product library: each arg is NAME=FLAGS, e.g.
# q4="-DFM_QMINB=4"; builds _lib/var/lib_NAME.so (ptxas log beside it)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2005_03156_b200/_lib/var
rm -f paper_2005_03156_b200/_lib/var/*.so paper_2005_03156_b200/_lib/var/*.log
for v in "$@"; do
  N=${v%%=*}; F=${v#*=}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    $F -Xcompiler -fPIC,-O3,-ffp-contract=off,-pthread -shared \
    paper_2005_03156_b200/csrc/fastmap_b200.cu paper_2005_03156_b200/csrc/index_gpu.cu paper_2005_03156_b200/csrc/index_host.cpp \
    paper_2005_03156_b200/csrc/io.cpp paper_2005_03156_b200/csrc/simple.cu paper_2005_03156_b200/csrc/multi.cu \
    -o paper_2005_03156_b200/_lib/var/lib_$N.so -Xptxas -v 2> paper_2005_03156_b200/_lib/var/ptxas_$N.log &
done
wait
for v in "$@"; do N=${v%%=*}; echo $N $(grep -A2 "Function properties for.*${KER:-resolve_quick_kernelILb0}" paper_2005_03156_b200/_lib/var/ptxas_$N.log | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores"); done
