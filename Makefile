# Build recipe for the B200 projection library, its workload generators and
# the CPU oracle.  `python -c "import __graft_entry__ as g; g.build()"` runs
# this.  The product is compiled for sm_100a only, with FMA contraction off
# on both the device (--fmad=false) and the host (-ffp-contract=off) sides.
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
CC        ?= gcc
REF       ?= /root/reference
PKG       := paper_2005_03156_b200
LIBDIR    := $(PKG)/_lib
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Xptxas -v \
             -Xcompiler -fPIC,-O3,-ffp-contract=off,-pthread
HOSTFLAGS := -O3 -fPIC -ffp-contract=off -pthread

PRODUCT_SRC := $(PKG)/csrc/fastmap_b200.cu $(PKG)/csrc/index_gpu.cu $(PKG)/csrc/index_host.cpp \
               $(PKG)/csrc/io.cpp $(PKG)/csrc/simple.cu $(PKG)/csrc/multi.cu
PRODUCT_HDR := include/fastmap_b200.h $(PKG)/csrc/index_format.h \
               $(PKG)/csrc/index_build.h $(PKG)/csrc/query.cuh $(PKG)/csrc/sweep.h \
               $(PKG)/csrc/record_encode.h $(PKG)/csrc/hierarchy.h $(PKG)/csrc/binned.cuh

all: product synth oracle ref

product: $(LIBDIR)/libfastmap_b200.so
synth: $(LIBDIR)/libfastmap_synth.so
oracle: oracle/liboracle.so

$(LIBDIR)/libfastmap_b200.so: $(PRODUCT_SRC) $(PRODUCT_HDR)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -shared $(PRODUCT_SRC) -o $@ 2> $(LIBDIR)/ptxas.log || (cat $(LIBDIR)/ptxas.log; exit 1)
	@grep -E "registers|spill" $(LIBDIR)/ptxas.log | sed 's/^/  /' | head -20

# workload generators: host (synth.cpp) and device (synth_gpu.cu) streams
# share synth_rng.h; both sides without FMA contraction
$(LIBDIR)/libfastmap_synth.so: $(PKG)/csrc/synth.cpp $(PKG)/csrc/synth_gpu.cu $(PKG)/csrc/synth_rng.h
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -O3 --fmad=false -std=c++17 -Xcompiler -fPIC,-O3,-ffp-contract=off,-pthread \
	  -shared $(PKG)/csrc/synth.cpp $(PKG)/csrc/synth_gpu.cu -o $@

oracle/liboracle.so: oracle/oracle.c oracle/Makefile
	$(MAKE) --no-print-directory -f oracle/Makefile $(CURDIR)/oracle/liboracle.so

# reference-compiled oracle: the unmodified reference headers, read in place
ref: product
	@if [ -d "$(REF)/proj/include/fastmap" ]; then \
	  $(MAKE) --no-print-directory oracle/_ref/libfastmap_ref.so oracle/_ref/adapter_check; \
	else echo "reference sources absent: using prebuilt oracle/_ref (if any)"; fi

oracle/_ref/libfastmap_ref.so: oracle/ref_shim.cpp oracle/Makefile
	$(MAKE) --no-print-directory -f oracle/Makefile REF=$(REF) $(CURDIR)/oracle/_ref/libfastmap_ref.so

# the C++ drop-in adapter compiled against the reference's own headers
oracle/_ref/adapter_check: tests/cpp/adapter_check.cpp include/fastmap_b200/fastmap_gpu.hpp include/fastmap_b200.h $(LIBDIR)/libfastmap_b200.so
	@mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O2 -ffp-contract=off -I$(REF)/proj/include -Iinclude $< \
	  -L$(LIBDIR) -lfastmap_b200 -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' -o $@

clean:
	rm -rf $(LIBDIR) oracle/liboracle.so oracle/_ref

.PHONY: all product synth oracle ref clean
