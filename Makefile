# Builds the product library (sm_100a device code + host C++) and the test oracle.
# The kernel translation units (native K = 1 and K = 2-4, each per ticks-per-block NT; exact) and the
# host code compile in parallel (make -j).
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
NATIVE_OBJS = $(LIBDIR)/kernels_native_k1_nt8.o $(LIBDIR)/kernels_native_k1_nt16.o \
              $(LIBDIR)/kernels_native_kn_nt4.o $(LIBDIR)/kernels_native_kn_nt16.o
NATIVE64_OBJS = $(LIBDIR)/kernels_native64_scan_k1_ln0.o $(LIBDIR)/kernels_native64_scan_k1_ln1.o \
                $(LIBDIR)/kernels_native64_scan_kn_ln0.o $(LIBDIR)/kernels_native64_scan_kn_ln1.o \
                $(LIBDIR)/kernels_native64_free.o
OBJS = $(LIBDIR)/bbe_sim.o $(NATIVE_OBJS) $(NATIVE64_OBJS) $(LIBDIR)/kernels_exact.o $(LIBDIR)/host_mt.o

all: $(LIB) oracle

$(LIBDIR)/bbe_sim.o: $(CSRC)/bbe_sim.cu $(COMMON)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(LIBDIR)/ptxas_host.log || (cat $(LIBDIR)/ptxas_host.log; exit 1)

# native kernels: one object per (K half, ticks per block NT)
NATIVE_DEPS = $(CSRC)/kernels_native.cu $(CSRC)/native_kernel.cuh $(COMMON)
$(LIBDIR)/kernels_native_k1_nt%.o: $(NATIVE_DEPS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -DBBE_NATIVE_K1 -DBBE_NATIVE_NT=$* -c -o $@ $< 2> $(LIBDIR)/ptxas_native_k1_nt$*.log || (cat $(LIBDIR)/ptxas_native_k1_nt$*.log; exit 1)

$(LIBDIR)/kernels_native_kn_nt%.o: $(NATIVE_DEPS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -DBBE_NATIVE_NT=$* -c -o $@ $< 2> $(LIBDIR)/ptxas_native_kn_nt$*.log || (cat $(LIBDIR)/ptxas_native_kn_nt$*.log; exit 1)

# NATIVE64 kernels: with and without the front-runner scan
NATIVE64_DEPS = $(CSRC)/kernels_native64.cu $(CSRC)/native64_kernel.cuh $(COMMON)
$(LIBDIR)/kernels_native64_scan_k1_ln%.o: $(NATIVE64_DEPS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -DBBE_N64_SCAN=1 -DBBE_N64_K1=1 -DBBE_N64_LN=$* -c -o $@ $< 2> $(LIBDIR)/ptxas_native64_scan_k1_ln$*.log || (cat $(LIBDIR)/ptxas_native64_scan_k1_ln$*.log; exit 1)

$(LIBDIR)/kernels_native64_scan_kn_ln%.o: $(NATIVE64_DEPS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -DBBE_N64_SCAN=1 -DBBE_N64_K1=0 -DBBE_N64_LN=$* -c -o $@ $< 2> $(LIBDIR)/ptxas_native64_scan_kn_ln$*.log || (cat $(LIBDIR)/ptxas_native64_scan_kn_ln$*.log; exit 1)

$(LIBDIR)/kernels_native64_free.o: $(NATIVE64_DEPS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -DBBE_N64_SCAN=0 -c -o $@ $< 2> $(LIBDIR)/ptxas_native64_free.log || (cat $(LIBDIR)/ptxas_native64_free.log; exit 1)

$(LIBDIR)/kernels_exact.o: $(CSRC)/kernels_exact.cu $(CSRC)/exact_kernel.cuh $(CSRC)/mt_stream.cuh $(COMMON)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(LIBDIR)/ptxas_exact.log || (cat $(LIBDIR)/ptxas_exact.log; exit 1)

$(LIBDIR)/host_mt.o: $(CSRC)/host_mt.cpp
	@mkdir -p $(LIBDIR)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -ldl
	@cat $(LIBDIR)/ptxas_native_k1_nt*.log $(LIBDIR)/ptxas_native_kn_nt*.log $(LIBDIR)/ptxas_native64_*.log $(LIBDIR)/ptxas_exact.log > $(LIBDIR)/ptxas.log

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIB) $(LIBDIR)/*.o $(LIBDIR)/*.log
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
