# libmcf.so (sm_100a) + the CPU oracle.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
PKG := paper_1108_2580_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr

all: $(PKG)/libmcf.so oracle

# ptxas -v output (registers / spills per kernel) goes to build/ptxas.log
$(PKG)/libmcf.so: $(SRC) $(PKG)/csrc/common.cuh include/mcf.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -ldl 2> build/ptxas.log || (cat build/ptxas.log; false)

# micro-benchmarks used for the roofline peaks (profiles/fp32_peak.json)
MICRO := $(patsubst %.cu,%,$(wildcard tools/micro/*.cu))
micro: $(MICRO)
tools/micro/%: tools/micro/%.cu
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o $@ $<

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(PKG)/libmcf.so oracle/liboracle.so

.PHONY: all oracle clean micro
