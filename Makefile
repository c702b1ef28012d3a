# libmcf.so (sm_100a) + the CPU oracle.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
PKG := paper_1108_2580_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr

all: $(PKG)/libmcf.so oracle

$(PKG)/libmcf.so: $(SRC) $(PKG)/csrc/common.cuh include/mcf.h
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; false)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(PKG)/libmcf.so oracle/liboracle.so

.PHONY: all oracle clean
