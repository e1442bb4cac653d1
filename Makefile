# Builds the product library (sm_100a device code + host C++) and the test oracle.
# The kernel translation units (native K = 1, native K = 2-4, exact) and the host code compile in
# parallel (make -j).
NVCC ?= nvcc
CXX ?= g++
ARCH = -gencode arch=compute_100a,code=sm_100a
NVEXTRA ?=
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v $(NVEXTRA)
CXXFLAGS = -O3 -std=c++17 -fPIC
LIBDIR ?= paper_2108_02419_b200/_lib
LIB = $(LIBDIR)/libbbe_sim.so
CSRC = paper_2108_02419_b200/csrc
COMMON = $(CSRC)/common.cuh $(CSRC)/kernels.h include/bbe_sim.h
OBJS = $(LIBDIR)/bbe_sim.o $(LIBDIR)/kernels_native_k1.o $(LIBDIR)/kernels_native.o $(LIBDIR)/kernels_exact.o \
       $(LIBDIR)/host_mt.o

all: $(LIB) oracle

$(LIBDIR)/bbe_sim.o: $(CSRC)/bbe_sim.cu $(COMMON)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(LIBDIR)/ptxas_host.log || (cat $(LIBDIR)/ptxas_host.log; exit 1)

$(LIBDIR)/kernels_native_k1.o: $(CSRC)/kernels_native.cu $(CSRC)/native_kernel.cuh $(COMMON)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -DBBE_NATIVE_K1 -c -o $@ $< 2> $(LIBDIR)/ptxas_native_k1.log || (cat $(LIBDIR)/ptxas_native_k1.log; exit 1)

$(LIBDIR)/kernels_native.o: $(CSRC)/kernels_native.cu $(CSRC)/native_kernel.cuh $(COMMON)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(LIBDIR)/ptxas_native.log || (cat $(LIBDIR)/ptxas_native.log; exit 1)

$(LIBDIR)/kernels_exact.o: $(CSRC)/kernels_exact.cu $(CSRC)/exact_kernel.cuh $(CSRC)/mt_stream.cuh $(COMMON)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(LIBDIR)/ptxas_exact.log || (cat $(LIBDIR)/ptxas_exact.log; exit 1)

$(LIBDIR)/host_mt.o: $(CSRC)/host_mt.cpp
	@mkdir -p $(LIBDIR)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -ldl
	@cat $(LIBDIR)/ptxas_native_k1.log $(LIBDIR)/ptxas_native.log $(LIBDIR)/ptxas_exact.log > $(LIBDIR)/ptxas.log

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIB) $(LIBDIR)/*.o $(LIBDIR)/*.log
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
