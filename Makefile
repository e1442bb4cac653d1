# Builds the product library (sm_100a device code + host C++) and the test oracle.
NVCC ?= nvcc
CXX ?= g++
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v
CXXFLAGS = -O3 -std=c++17 -fPIC
LIBDIR = paper_2108_02419_b200/_lib
LIB = $(LIBDIR)/libbbe_sim.so
CSRC = paper_2108_02419_b200/csrc
CU_DEPS = $(CSRC)/bbe_sim.cu $(wildcard $(CSRC)/*.cuh) include/bbe_sim.h

all: $(LIB) oracle

$(LIBDIR)/bbe_sim.o: $(CU_DEPS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/bbe_sim.cu 2> $(LIBDIR)/ptxas.log || (cat $(LIBDIR)/ptxas.log; exit 1)

$(LIBDIR)/host_mt.o: $(CSRC)/host_mt.cpp
	@mkdir -p $(LIBDIR)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(LIB): $(LIBDIR)/bbe_sim.o $(LIBDIR)/host_mt.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -ldl

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIB) $(LIBDIR)/*.o
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
