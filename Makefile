# Builds the product library (sm_100a) and the test oracle.
NVCC ?= nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
          --expt-relaxed-constexpr -Xptxas -v
LIB = paper_2108_02419_b200/_lib/libbbe_sim.so
SRC = paper_2108_02419_b200/csrc/bbe_sim.cu $(wildcard paper_2108_02419_b200/csrc/*.cuh) include/bbe_sim.h

all: $(LIB) oracle

$(LIB): $(SRC)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -o $@ paper_2108_02419_b200/csrc/bbe_sim.cu -ldl 2> paper_2108_02419_b200/_lib/ptxas.log || (cat paper_2108_02419_b200/_lib/ptxas.log; exit 1)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
